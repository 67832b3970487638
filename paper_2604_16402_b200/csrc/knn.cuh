// kNN engine shared by pass 1 (per-bucket slabs), pass 2 (global) and insert
// candidate generation: screen + exact f64 rerank.
#pragma once
#include <vector>

#include <cuda_bf16.h>

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

// Brute-force mode of the tcgen05 screen (knn_tc.cu k_knn_screen_tc<true>).
struct TcBf {
  const float* qnorm = nullptr;    // [ntile * 128] |q|^2 of the sorted query rows
  const float* qlo = nullptr;      // [ntile * 128] f32 bounds (lo > hi: no range)
  const float* qhi = nullptr;
  const uint32_t* span = nullptr;  // [ntile][2] phys column span of each query tile
  uint32_t S = 1;                  // column splits (CTAs) per tile
  uint64_t* keys = nullptr;        // [ntile * S][128][KP] heap entries, root = kept max, ~0 = empty
};
// keys per (query tile, split) of the split-BF16 screen of the sorted query
// rows q_hi / q_lo ([ntile * 128] x kp) against the index's live columns
// (masked_norms: |x|^2 per phys row, +inf for rows that are not live, padded to
// a whole column tile past phys_cap plus one: div_up(phys_cap, 64) * 64 + 64)
// x_hi / x_lo: the same split of the phys rows ([phys_cap] x kp)
void bf_screen_tc(const DevIndex& ix, const __nv_bfloat16* q_hi, const __nv_bfloat16* q_lo, const __nv_bfloat16* x_hi,
                  const __nv_bfloat16* x_lo, uint32_t ntile, const float* masked_norms, uint32_t KP, TcBf bf,
                  cudaStream_t st);
uint32_t tc_pad_cols();

// tcgen05 split-BF16 screen (knn_tc.cu): same output contract as the SIMT screen
// (per query row, KP candidate phys ids in cand[row * KP ..]).
bool knn_tc_supported(const DevIndex& ix, uint32_t KP);
void knn_screen_tc(const DevIndex& ix, const float* norms, const KnnJob* djobs, uint32_t njobs, uint32_t KP,
                   uint32_t* cand, bool causal, cudaStream_t st);

}  // namespace grab
