// kNN engine shared by pass 1 (per-bucket slabs), pass 2 (global) and insert
// candidate generation: screen + exact f64 rerank.
#pragma once
#include <vector>

#include "index.cuh"

namespace grab {

constexpr uint32_t kKnnBM = 128;  // query rows per job / CTA

// rows [r0, r0+nr) (phys) against candidate phys range [c0, c1)
struct KnnJob {
  uint32_t r0, nr, c0, c1;
};

// For every query row p of every job: out_ids[p*K + j] / out_d[p*K + j] = the
// K nearest valid candidates (excluding p itself), ascending by (f64 dist,
// tiebreak) where tiebreak = slot (tb_slot) or phys (slab-local column order).
// Unfilled entries stay as initialised by the caller (SENTINEL).
// causal: only candidates c < row (same slab => slot order), as the insert's
// in-bucket candidates (updater.py:143).
void knn_device(const DevIndex& ix, const float* norms, const std::vector<KnnJob>& jobs, uint32_t K, bool tb_slot,
                uint32_t* out_ids, double* out_d, cudaStream_t st, bool causal = false);
void row_norms(const DevIndex& ix, float* out, cudaStream_t st);

// tcgen05 split-BF16 screen (knn_tc.cu): same output contract as the SIMT screen
// (per query row, KP candidate phys ids in cand[row * KP ..]).
bool knn_tc_supported(const DevIndex& ix, uint32_t KP);
void knn_screen_tc(const DevIndex& ix, const float* norms, const KnnJob* djobs, uint32_t njobs, uint32_t KP,
                   uint32_t* cand, bool causal, cudaStream_t st);

}  // namespace grab
