// bucket_select: range -> inclusive bucket interval, and per-scalar bucket ids.
// Reference: bucket_ids_of / bucket_of / intersecting_buckets (layout.py:157-174).
// Bounds are rounded to f32 first (numpy 2 NEP-50 weak-float semantics of the
// reference's np.array([s], dtype=float32)); comparisons are in f32.
#include "index.cuh"

namespace grab {

__global__ void k_bucket_ids(const float* bound, uint32_t m, const float* s, uint64_t n, int32_t* out) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = bucket_of_f32(bound, m, s[i]);
}

__global__ void k_bucket_select(const float* bound, uint32_t m, const double* lo, const double* hi, uint64_t n,
                                int32_t* out_lo, int32_t* out_hi) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  out_lo[i] = bucket_of_f32(bound, m, __double2float_rn(lo[i]));
  out_hi[i] = bucket_of_f32(bound, m, __double2float_rn(hi[i]));
}

void launch_bucket_ids(const DevIndex& ix, const float* s, uint64_t n, int32_t* out, cudaStream_t st) {
  if (!n) return;
  k_bucket_ids<<<(unsigned)div_up(n, 256), 256, 0, st>>>(ix.bound, ix.m, s, n, out);
  GRAB_CHECK_LAUNCH();
}

void launch_bucket_select(const DevIndex& ix, const double* lo, const double* hi, uint64_t n, int32_t* out_lo,
                          int32_t* out_hi, cudaStream_t st) {
  if (!n) return;
  k_bucket_select<<<(unsigned)div_up(n, 256), 256, 0, st>>>(ix.bound, ix.m, lo, hi, n, out_lo, out_hi);
  GRAB_CHECK_LAUNCH();
}

}  // namespace grab
