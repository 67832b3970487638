// Search kernel arguments (filtered_beam_search + seed_sample).
#pragma once
#include <stdint.h>

#include "index.cuh"

namespace grab {

struct SearchArgs {
  // index (phys space)
  const float* X;
  const Attr* attr;
  const uint32_t* adj;
  const Attr* adja;  // per-adjacency-entry {scalar, slot} (DevIndex::adja)
  uint32_t dp, k_max;
  const float* bound;
  uint32_t m;
  const uint32_t* bstart;
  const uint32_t* bcount;
  const uint64_t* bcum;
  uint64_t n_live;
  // queries (rows padded to dp)
  const float* Q;
  const uint32_t* qphys;  // optional: query i = X row qphys[i] (insert candidate search)
  const double* lower;
  const double* upper;
  uint64_t range_stride;
  const uint64_t* seeds;
  uint64_t seed_base, ordinal0;
  uint32_t k, itopk, width, max_iter, want;
  // work list / overflow retry
  const uint32_t* qmap;
  uint32_t nwork;
  const uint32_t* nwork_dev;  // if set, the work count is read on the device
  uint32_t* gtab;
  uint32_t* ovf_list;
  uint32_t* ovf_count;
  // if set, warps claim work items dynamically (atomicAdd) instead of the static
  // stride: queries differ in cost, so this evens out the grid's tail
  uint32_t* work_ctr;
  // outputs (indexed by query id)
  int64_t* out_slots;
  double* out_dists;
  uint32_t* out_counts;
  grab_search_stats* out_stats;
};

struct SearchShape {
  uint32_t itopk, width, cmax, dsz, vlog2;
  // per-warp shared-memory layout (byte offsets, filled by make_shape)
  uint32_t o_qe, o_cd, o_cs, o_cp, o_dd, o_fr, o_q, warp_bytes, qbytes;
};

SearchShape make_shape(uint32_t itopk, uint32_t width, uint32_t k_max, uint32_t want, uint32_t max_iter, bool worst,
                       uint32_t dp, uint64_t live_rows, bool stats, uint64_t phys_rows);
void run_search(const DevIndex& ix, SearchArgs a, cudaStream_t st);

}  // namespace grab
