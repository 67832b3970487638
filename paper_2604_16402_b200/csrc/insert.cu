// placeholder until the insert pipeline lands
#include "ops.cuh"
namespace grab {
void insert_batch_device(DevIndex&, const float*, const float*, const int64_t*, uint64_t, uint32_t, uint32_t,
                         grab_insert_report*) {
  throw Error(GRAB_ERR_STATE, "insert not implemented yet");
}
void select_neighbors_device(const float*, uint64_t, uint32_t, int64_t, const int64_t*, const double*, const uint8_t*,
                             uint32_t, uint32_t, double, int64_t*, uint32_t*) {
  throw Error(GRAB_ERR_STATE, "nyi");
}
void try_rewire_device(const float*, uint64_t, uint32_t, uint32_t*, uint32_t, uint32_t, uint32_t, double, double,
                       uint32_t, int32_t*, int32_t*) {
  throw Error(GRAB_ERR_STATE, "nyi");
}
}  // namespace grab
