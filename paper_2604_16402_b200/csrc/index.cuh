// Device-resident GRAB index: bucket-slab physical layout + slot maps.
//
// Reference state (layout.py:22-104, 226-257): VectorStore X/scalars/ids in
// slot order, adjacency u32[N_cap x K_max] in slot ids, BucketMeta boundaries +
// M_I2B + M_B2I (members of each bucket in insertion = ascending-slot order).
//
// B200 layout: rows are physically grouped into one contiguous slab per bucket
// (members in M_B2I order, slab start 32-row aligned, d padded to a multiple of
// 4 floats so every row is a run of 16-byte vectors). A range predicate becomes
// the slab interval [bstart[lo], bstart[hi] + bcount[hi]); seed draw `flat`
// maps to phys = bstart[b] + offset with no list indirection; pass-1 kNN tiles
// are contiguous slabs. Adjacency is stored in PHYS ids so a gather needs no
// translation; Attr{scalar, slot} per phys row gives the pre-check value and
// the slot id for (dist, slot) tie-breaks in one 8-byte load.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <memory>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace grab {

struct DevIndex {
  int device = 0;
  int num_sms = 148;
  uint32_t dim = 0, dp = 0;  // dp = round_up(dim, 4)
  uint64_t n_cap = 0;        // slot capacity (N_cap)
  grab_build_params params{};
  cudaStream_t stream = nullptr;

  uint64_t count = 0;  // published live slots
  bool built = false;  // meta present

  // slot space
  uint32_t* slot2phys = nullptr;  // [n_cap]
  int32_t* i2b = nullptr;         // [n_cap], -1 unclaimed
  std::vector<int64_t> ids;       // store.ids (host, not on any hot path)

  // phys space
  uint64_t phys_cap = 0;  // rows allocated
  float* X = nullptr;     // [phys_cap x dp]
  Attr* attr = nullptr;   // [phys_cap]
  uint32_t* adj = nullptr;  // [phys_cap x k_max], phys ids
  // Search-side mirror of the adjacency: adja[p*K + j] = attr[adj[p*K + j]]
  // ({NaN, kNoSlot} for SENTINEL), so one coalesced row load gives every
  // neighbour's pre-check scalar and slot without a random 8-byte gather per
  // neighbour. Rebuilt lazily by the search path when adj_version moved.
  uint64_t adj_version = 1;  // bumped by every adjacency / layout mutation
  mutable Attr* adja = nullptr;
  // per-stream search scratch (visited tables, overflow list), grown on demand
  // and reused by later calls on the same stream (search.cu)
  std::shared_ptr<struct SearchWsCache> search_ws;
  mutable uint64_t adja_rows = 0, adja_version = 0;
  // guards adja; `ready` is recorded after a rebuild so searches on other
  // streams wait for it instead of reading a half-filled mirror
  struct AdjaSync {
    std::mutex mu;
    cudaEvent_t ready = nullptr;
    ~AdjaSync() {
      if (ready) cudaEventDestroy(ready);
    }
  };
  std::shared_ptr<AdjaSync> adja_sync = std::make_shared<AdjaSync>();

  // buckets
  uint32_t m = 0;
  uint32_t m_alloc = 0;        // bucket count the device tables below are sized for
  float* bound = nullptr;      // [m+1]
  uint32_t* bstart = nullptr;  // [m]
  uint32_t* bcount = nullptr;  // [m]
  uint64_t* bcum = nullptr;    // [m+1] prefix of bcount (seed draws)
  std::vector<float> h_bound;
  std::vector<uint32_t> h_bstart, h_bcount, h_bcap;

  std::vector<uint32_t> last_rewired;

  uint32_t k_max() const { return params.k_max; }
  size_t device_bytes() const;
};

// ---- upload.cu ----
// host -> device copy of a (large, pageable) host buffer, stream-ordered on st;
// the source may be reused as soon as the call returns
void upload_h2d(void* dst, const void* src, size_t bytes, cudaStream_t st);

// ---- layout.cu ----
void index_alloc_slots(DevIndex& ix);
void index_free(DevIndex& ix);
// (re)build ix.adja if the adjacency changed since the last search (search.cu)
void ensure_adja(const DevIndex& ix, cudaStream_t st);
void free_search_ws(DevIndex& ix);
// Lay out `count` slots whose bucket ids are in ix.i2b (device) and whose
// vectors/scalars are given in slot order (device pointers, rows of `dim`).
// Members of a bucket are ordered by ascending slot. Allocates slabs with
// headroom, fills X/attr/slot2phys, leaves adjacency SENTINEL.
void layout_from_slots(DevIndex& ix, const float* X_slot, const float* S_slot, uint64_t count,
                       const std::vector<uint32_t>& bucket_sizes);
// Append `b` fresh slots [start, start+b) (bucket ids already in ix.i2b) to
// their slabs, relayouting all slabs when one overflows.
void append_batch_device(DevIndex& ix, const float* vectors, const float* scalars, const int64_t* ids, uint64_t b,
                         uint32_t mem, uint64_t* start_out, uint64_t* end_out);
void layout_append(DevIndex& ix, const float* X_new, const float* S_new, uint64_t start, uint64_t b);
void upload_bucket_tables(DevIndex& ix);
// slot-space adjacency -> phys-space (import) and back (export)
void adjacency_slot_to_phys(DevIndex& ix, const uint32_t* adj_slot_dev, uint64_t n);
void adjacency_phys_to_slot(const DevIndex& ix, uint32_t* adj_slot_dev, uint64_t start, uint64_t n);
void gather_slot_rows(const DevIndex& ix, float* X_out_dev, float* S_out_dev, uint64_t start, uint64_t n);

// ---- bucket lookup (select.cu) ----
void launch_bucket_ids(const DevIndex& ix, const float* s, uint64_t n, int32_t* out, cudaStream_t st);
// partition_buckets edges (np.unique applied) for n device scalars (build.cu)
std::vector<float> partition_edges_device(const float* S, uint64_t n, uint32_t target, int strategy,
                                          cudaStream_t st);
void launch_bucket_select(const DevIndex& ix, const double* lo, const double* hi, uint64_t n,
                          int32_t* out_lo, int32_t* out_hi, cudaStream_t st);

// Device helper shared by kernels: count of interior edges <= s, i.e.
// searchsorted(boundaries[1:-1], s, 'right') (layout.py:157-160).
__device__ __forceinline__ int32_t bucket_of_f32(const float* bound, uint32_t m, float s) {
  int32_t lo = 0, hi = (int32_t)m - 1;  // interior edges bound[1..m-1]
  while (lo < hi) {
    int32_t mid = (lo + hi) >> 1;
    if (__ldg(bound + 1 + mid) <= s)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

}  // namespace grab
