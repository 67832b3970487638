// kNN screen on the 5th-gen tensor cores (tcgen05 + TMEM + TMA), sm_100a.
//
// Reference: pairwise_sq_dists + topk_ids_by_distance (builder.py:79-113) --
// the build's only dense contraction (pass-1 buckets, the global graph and the
// insert's in-bucket candidates all go through knn_device()).
//
// dot(a, b) is computed as a split-BF16 product: x = hi + lo with
// hi = bf16(x), lo = bf16(x - hi); a.b ~= ah.bh + ah.bl + al.bh (three UMMAs
// into one fp32 TMEM accumulator) -- relative error ~1e-5, far below the gap
// between a row's k-th and (k+16)-th neighbour, and every survivor is
// re-ranked exactly in f64 afterwards (knn.cu k_knn_rerank).
//
// CTA = one 128-row query tile x a stream of 64-row candidate tiles:
//   warp 0    TMA producer (A hi/lo once, B hi/lo through a 3-stage ring)
//   warp 1    TMEM allocator + single-thread UMMA issuer
//             (kind::f16, BF16 in, F32 accumulate, M=128 N=64 K=16)
//   warps 2-5 epilogue: tcgen05.ld 32x32b (thread t owns TMEM lane t = query
//             row t), d = |a|^2 + |b|^2 - 2 a.b, per-row max-heap of K+16
// Two TMEM accumulator stages let the MMA of tile i+1 overlap the epilogue of
// tile i.
#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "knn.cuh"

namespace grab {

namespace tc {

constexpr uint32_t BM = 128, BN = 64, KCH = 64;  // KCH: bf16 per 128-byte swizzle row
constexpr uint32_t MAX_STAGES = 3;
constexpr uint32_t KP_MAX = 80;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int32_t x, int32_t y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(x), "r"(y)
      : "memory");
}

// K-major, 128-byte swizzle UMMA shared-memory descriptor (SM100 layout):
// start>>4 [0,14), LBO>>4 [16,30) (unused for swizzled K-major), SBO>>4 [32,46)
// = 1024 B between 8-row groups, version 1 at [46,48), layout 2 (SWIZZLE_128B) at [61,64).
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr & 0x3FFFF) >> 4);
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// kind::f16 instruction descriptor: F32 accumulate, BF16 A/B, K-major, M=128, N=64
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((BN >> 3) << 17) | ((BM >> 4) << 24);

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(kIdesc), "r"(accumulate));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

// Max-heap of n keys for one row, element i at h[i * BM] (rows interleaved so
// the 32 lanes of a warp touch 32 consecutive words: no bank conflicts).
// HEAP_ARY-ary (4): half the levels of a binary heap, and a level's child loads
// are independent, so the sift-down's chain of dependent shared loads halves
// (screen 47 -> 38 ms at cfg2 pass 1)
#ifndef GRAB_HEAP_ARY
#define GRAB_HEAP_ARY 4
#endif
__device__ __forceinline__ void heap_replace_top(uint64_t* h, uint32_t n, uint64_t key) {
  constexpr uint32_t A = GRAB_HEAP_ARY;
  uint32_t i = 0;
  while (true) {
    const uint32_t c0 = A * i + 1;
    if (c0 >= n) break;
    uint64_t kb = h[c0 * BM];
    uint32_t big = c0;
#pragma unroll
    for (uint32_t j = 1; j < A; ++j) {
      const uint32_t c = c0 + j;
      const uint64_t v = c < n ? h[c * BM] : 0ull;
      if (v > kb) {
        kb = v;
        big = c;
      }
    }
    if (kb <= key) break;
    h[i * BM] = kb;
    i = big;
  }
  h[i * BM] = key;
}

struct Smem {
  // all operand tiles are 1024-byte aligned (128B swizzle atom = 8 x 128 B)
  static constexpr uint32_t kChunkA = BM * 128;  // one 64-bf16 K-chunk of the A tile
  static constexpr uint32_t kChunkB = BN * 128;
};

constexpr uint32_t kThreads = 320;  // TMA warp, MMA warp, 8 epilogue warps

// BF = true: the batched brute-force screen (bf_screen_tc). The A tile is 128
// range queries (sorted by slab start, tmap over their hi/lo split), the B
// stream is the phys columns of the tile's span [span[2t], span[2t+1]) split
// S ways (CTA (t, s) takes column tiles s, s+S, ...), every column is checked
// against the row's own f32 range, and the CTA writes each row's raw heap
// (root = the kept maximum, ~0 = empty) to keys[(cta * BM + row) * KP ..].
template <bool BF>
__global__ void __launch_bounds__(kThreads, 1)
    k_knn_screen_tc(const __grid_constant__ CUtensorMap tmap_ahi, const __grid_constant__ CUtensorMap tmap_alo,
                    const __grid_constant__ CUtensorMap tmap_bhi, const __grid_constant__ CUtensorMap tmap_blo,
                    const KnnJob* jobs, const Attr* attr, const float* row_norms, const float* norms,
                    uint32_t nkc, uint32_t KP, uint32_t* cand, int causal, uint32_t STAGES, uint32_t NG,
                    int stream_a, const TcBf bf) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // aligned by an offset from the shared array (not an integer round trip), so
  // the compiler keeps the shared address space: the heaps compile to LDS/STS,
  // not generic loads with an address-space conversion each
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  // resident A (d <= 128): A hi/lo for every K chunk loaded once, the ring holds
  // one column tile's B hi/lo (all K chunks) per stage. Streamed A (d > 128):
  // every ring stage holds ONE K chunk of A hi/lo and B hi/lo, so any d fits and
  // the accumulator sums the chunks in TMEM.
  const uint32_t a_bytes = stream_a ? 0u : nkc * Smem::kChunkA;  // resident A per hi / lo
  const uint32_t b_bytes = stream_a ? 0u : nkc * Smem::kChunkB;
  const uint32_t st_bytes = stream_a ? 2 * (Smem::kChunkA + Smem::kChunkB) : 2 * b_bytes;  // one ring stage
  uint8_t* A_hi = smem;
  uint8_t* A_lo = A_hi + a_bytes;
  uint8_t* B = A_lo + a_bytes;  // STAGES x stage
  uint64_t* H = (uint64_t*)(B + STAGES * st_bytes);  // NG column groups x [KP][BM]
  uint64_t* bars = H + NG * BM * KP;
  uint64_t* a_full = bars;
  uint64_t* b_full = bars + 1;
  uint64_t* b_empty = b_full + MAX_STAGES;
  uint64_t* acc_full = b_empty + MAX_STAGES;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = (uint32_t*)(acc_empty + 2);

  uint32_t r0, nr, c0, c1, split = 0, S = 1;
  if constexpr (BF) {
    const uint32_t tile = blockIdx.x / bf.S;
    split = blockIdx.x % bf.S;
    S = bf.S;
    r0 = tile * BM;
    nr = BM;
    c0 = bf.span[2 * tile];
    c1 = bf.span[2 * tile + 1];
    if (c1 < c0) c1 = c0;  // no live query in the tile
  } else {
    const KnnJob job = jobs[blockIdx.x];
    r0 = job.r0;
    nr = job.nr;
    c0 = job.c0;
    c1 = job.c1;
  }
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t nct = (c1 - c0 + BN - 1) / BN;  // column tiles of the span
  const uint32_t ntiles = nct > split ? (nct - split + S - 1) / S : 0;  // this CTA's share
  // first column of this CTA's t-th column tile
  auto col_of = [&](uint32_t t) -> uint32_t { return c0 + (split + t * S) * BN; };

  if (threadIdx.x == 0) {
    mbar_init(a_full, 1);
    for (uint32_t s = 0; s < STAGES; ++s) {
      mbar_init(b_full + s, 1);
      mbar_init(b_empty + s, 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(acc_full + s, 1);
      mbar_init(acc_empty + s, 4 * NG);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(2 * BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (uint32_t i = threadIdx.x; i < NG * BM * KP; i += blockDim.x) H[i] = ~0ull;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0 && stream_a) {
    if (lane == 0) {
      // ---- TMA producer, streamed A: ring slot u = (tile t, K chunk c)
      uint32_t u = 0;
      for (uint32_t t = 0; t < ntiles; ++t) {
        const int32_t row = (int32_t)col_of(t);
        for (uint32_t c = 0; c < nkc; ++c, ++u) {
          const uint32_t s = u % STAGES, round = u / STAGES;
          mbar_wait(b_empty + s, (round & 1) ^ 1);
          uint8_t* ah = B + s * st_bytes;
          uint8_t* al = ah + Smem::kChunkA;
          uint8_t* bh = al + Smem::kChunkA;
          uint8_t* bl = bh + Smem::kChunkB;
          mbar_expect_tx(b_full + s, st_bytes);
          tma_load_2d(ah, &tmap_ahi, b_full + s, (int32_t)(c * KCH), (int32_t)r0);
          tma_load_2d(al, &tmap_alo, b_full + s, (int32_t)(c * KCH), (int32_t)r0);
          tma_load_2d(bh, &tmap_bhi, b_full + s, (int32_t)(c * KCH), row);
          tma_load_2d(bl, &tmap_blo, b_full + s, (int32_t)(c * KCH), row);
        }
      }
    }
  } else if (warp == 1 && stream_a) {
    if (lane == 0) {
      // ---- UMMA issuer, streamed A: one commit per K chunk frees its ring slot
      uint32_t u = 0;
      for (uint32_t t = 0; t < ntiles; ++t) {
        const uint32_t as = t & 1, around = t >> 1;
        mbar_wait(acc_empty + as, (around & 1) ^ 1);
        const uint32_t d_tmem = tmem_base + as * BN;
        for (uint32_t c = 0; c < nkc; ++c, ++u) {
          const uint32_t s = u % STAGES, round = u / STAGES;
          mbar_wait(b_full + s, round & 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t ah = smem_u32(B + s * st_bytes), al = ah + Smem::kChunkA;
          const uint32_t bh = al + Smem::kChunkA, bl = bh + Smem::kChunkB;
#pragma unroll
          for (uint32_t kk = 0; kk < 4; ++kk) {
            const uint32_t off = kk * 32;
            umma_bf16(d_tmem, smem_desc(ah + off), smem_desc(bh + off), (c | kk) != 0u);
            umma_bf16(d_tmem, smem_desc(ah + off), smem_desc(bl + off), 1);
            umma_bf16(d_tmem, smem_desc(al + off), smem_desc(bh + off), 1);
          }
          umma_commit(b_empty + s);
        }
        umma_commit(acc_full + as);
      }
    }
  } else if (warp == 0) {
    if (lane == 0) {
      // ---- TMA producer
      mbar_expect_tx(a_full, 2 * a_bytes);
      for (uint32_t c = 0; c < nkc; ++c) {
        tma_load_2d(A_hi + c * Smem::kChunkA, &tmap_ahi, a_full, (int32_t)(c * KCH), (int32_t)r0);
        tma_load_2d(A_lo + c * Smem::kChunkA, &tmap_alo, a_full, (int32_t)(c * KCH), (int32_t)r0);
      }
      for (uint32_t t = 0; t < ntiles; ++t) {
        const uint32_t s = t % STAGES, round = t / STAGES;
        mbar_wait(b_empty + s, (round & 1) ^ 1);
        uint8_t* bh = B + s * 2 * b_bytes;
        uint8_t* bl = bh + b_bytes;
        mbar_expect_tx(b_full + s, 2 * b_bytes);
        const int32_t row = (int32_t)col_of(t);
        for (uint32_t c = 0; c < nkc; ++c) {
          tma_load_2d(bh + c * Smem::kChunkB, &tmap_bhi, b_full + s, (int32_t)(c * KCH), row);
          tma_load_2d(bl + c * Smem::kChunkB, &tmap_blo, b_full + s, (int32_t)(c * KCH), row);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---- UMMA issuer
      mbar_wait(a_full, 0);
      for (uint32_t t = 0; t < ntiles; ++t) {
        const uint32_t s = t % STAGES, round = t / STAGES;
        const uint32_t as = t & 1, around = t >> 1;
        mbar_wait(acc_empty + as, (around & 1) ^ 1);
        mbar_wait(b_full + s, round & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t d_tmem = tmem_base + as * BN;
        const uint32_t bh = smem_u32(B + s * 2 * b_bytes), bl = bh + b_bytes;
        const uint32_t ah = smem_u32(A_hi), al = smem_u32(A_lo);
        uint32_t acc = 0;
        for (uint32_t c = 0; c < nkc; ++c) {
#pragma unroll
          for (uint32_t kk = 0; kk < 4; ++kk) {  // 4 x K=16 bf16 = 128 B per swizzle row
            const uint32_t off = kk * 32;
            const uint64_t dah = smem_desc(ah + c * Smem::kChunkA + off);
            const uint64_t dal = smem_desc(al + c * Smem::kChunkA + off);
            const uint64_t dbh = smem_desc(bh + c * Smem::kChunkB + off);
            const uint64_t dbl = smem_desc(bl + c * Smem::kChunkB + off);
            umma_bf16(d_tmem, dah, dbh, acc);
            acc = 1;
            umma_bf16(d_tmem, dah, dbl, 1);
            umma_bf16(d_tmem, dal, dbh, 1);
          }
        }
        umma_commit(b_empty + s);     // smem stage reusable once these MMAs retire
        umma_commit(acc_full + as);   // accumulator ready for the epilogue
      }
    }
  } else {
    // ---- epilogue: warp w reads TMEM lanes 32*(w%4) .. +31 = query rows;
    // with NG = 2 two warps share a sub-partition, each owning half of every
    // tile's columns and a private heap per row (merged at the end).
    const uint32_t e = warp - 2, sub = warp & 3, grp = e >> 2;
    const uint32_t r = sub * 32 + lane;
    const uint32_t prow = r0 + r;
    const bool active = grp < NG;
    float qlo = 0.f, qhi = 0.f;
    bool row_ok;
    if constexpr (BF) {
      qlo = bf.qlo[prow];
      qhi = bf.qhi[prow];
      row_ok = active && qlo <= qhi;  // padding rows and empty ranges carry lo > hi
    } else {
      row_ok = active && r < nr && attr[prow].slot != kNoSlot;
    }
    const float a2 = row_ok ? (BF ? bf.qnorm[prow] : row_norms[prow]) : 0.f;
    uint64_t* h = H + grp * BM * KP + r;  // interleaved: element i at h[i * BM]
    uint64_t top = ~0ull;
    const uint32_t QN = 4 / NG;  // 16-column chunks per warp per tile
    for (uint32_t t = 0; active && t < ntiles; ++t) {
      const uint32_t as = t & 1, around = t >> 1;
      mbar_wait(acc_full + as, around & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t col0 = grp * QN * 16;
      const uint32_t taddr = tmem_base + ((sub * 32) << 16) + as * BN + col0;
      uint32_t v[4][16];
      tmem_ld16(taddr + 0, v[0]);
      tmem_ld16(taddr + 16, v[1]);
      if (QN == 4) {
        tmem_ld16(taddr + 32, v[2]);
        tmem_ld16(taddr + 48, v[3]);
      }
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) mbar_arrive(acc_empty + as);
      {  // every lane runs the chunk loop (the insertion pass below is warp-synchronous)
        const uint32_t cb = col_of(t) + col0;
        // |b|^2 with +inf for headroom rows / past the tile's end (one broadcast
        // float4 load per 4 columns); the heap key is only built for survivors
        // of an f32 threshold test against the current K'-th distance.
        // (<= FLT_MAX, not inf: a hit is always finite -- +inf norms never pass)
        const float thr = top == ~0ull ? 3.402823466e38f : __uint_as_float((uint32_t)(top >> 32));
        // admissible survivors of chunk q (finite, not the row itself, in range,
        // causal for insert candidates) among its threshold hits
        auto chunk_pend = [&](uint32_t q, uint32_t hit) -> uint32_t {
          uint32_t pend = 0;
          if constexpr (BF) {
            // the row's own range on the column's scalar: lane j loads column j's
            // scalar once and the 16 are shuffled to every row (lane); n_live /
            // headroom columns already carry +inf norms
            const uint32_t cl = cb + q * 16 + (lane & 15);
            const float scl = cl < c1 ? __ldg(&attr[cl].s) : __int_as_float(0x7FC00000);
#pragma unroll
            for (uint32_t j = 0; j < 16; ++j) {
              const float sc = __shfl_sync(0xFFFFFFFFu, scl, j);  // NaN past c1: fails both tests
              pend |= (uint32_t)(row_ok && ((hit >> j) & 1u) && sc >= qlo && sc <= qhi) << j;
            }
          } else {
            // the chunk's admissible columns as one mask: inside the job's span
            // (warp-uniform), not the row itself, and for causal jobs only
            // columns before the row
            const uint32_t cq = cb + q * 16;
            uint32_t m = c1 > cq ? (c1 - cq >= 16u ? 0xFFFFu : (1u << (c1 - cq)) - 1u) : 0u;
            if (prow >= cq && prow < cq + 16u) m &= ~(1u << (prow - cq));
            if (causal) m &= prow < cq ? 0u : (prow - cq >= 15u ? 0xFFFFu : (2u << (prow - cq)) - 1u);
            pend = row_ok ? (hit & m) : 0u;
          }
          return pend;
        };
        // chunks in pairs: one insertion loop per 32 columns, so a pass serves
        // the survivors of both chunks (the loop runs max-over-lanes survivors
        // of the pair instead of the sum of the two chunks' maxima)
#pragma unroll
        for (uint32_t qp = 0; qp < 2; ++qp) {
          if (2 * qp >= QN) break;
          // branch-free pass over 32 columns: distances + survivor masks
          float d[2][16];
          uint32_t hit[2] = {0u, 0u};
#pragma unroll
          for (uint32_t h2 = 0; h2 < 2; ++h2) {
            const uint32_t q = 2 * qp + h2;
#pragma unroll
            for (uint32_t j4 = 0; j4 < 4; ++j4) {
              const float4 n4 = __ldg(reinterpret_cast<const float4*>(norms + cb + q * 16) + j4);
              const float b2[4] = {n4.x, n4.y, n4.z, n4.w};
#pragma unroll
              for (uint32_t u = 0; u < 4; ++u) {
                const uint32_t j = 4 * j4 + u;
                d[h2][j] = fmaxf(fmaf(-2.f, __uint_as_float(v[q][j]), a2 + b2[u]), 0.f);
                hit[h2] |= (uint32_t)(d[h2][j] <= thr) << j;
              }
            }
          }
          if (!__any_sync(0xFFFFFFFFu, (hit[0] | hit[1]) != 0u)) continue;  // the common case after the first tiles
          uint32_t pend = 0;
          if (__any_sync(0xFFFFFFFFu, hit[0] != 0u)) pend = chunk_pend(2 * qp, hit[0]);
          if (__any_sync(0xFFFFFFFFu, hit[1] != 0u)) pend |= chunk_pend(2 * qp + 1, hit[1]) << 16;
          // heap insertions lane-parallel: every lane takes its NEXT survivor in
          // the same pass, so a pass costs one sift-down for all lanes at once
          // (a per-column loop would run one pass per distinct hit column);
          // per row the keys still arrive in column order
          while (__any_sync(0xFFFFFFFFu, pend != 0u)) {
            if (pend) {
              const uint32_t jb = __ffs(pend) - 1;
              pend &= pend - 1;
              // d[jb] by a binary select tree on jb's bits (31 selects, no compares)
              float t16[16], t8[8], t4[4];
#pragma unroll
              for (uint32_t i = 0; i < 16; ++i) t16[i] = (jb & 1u) ? d[i >> 3][((2 * i) & 15) + 1] : d[i >> 3][(2 * i) & 15];
#pragma unroll
              for (uint32_t i = 0; i < 8; ++i) t8[i] = (jb & 2u) ? t16[2 * i + 1] : t16[2 * i];
#pragma unroll
              for (uint32_t i = 0; i < 4; ++i) t4[i] = (jb & 4u) ? t8[2 * i + 1] : t8[2 * i];
              const float t2a = (jb & 8u) ? t4[1] : t4[0], t2b = (jb & 8u) ? t4[3] : t4[2];
              const float dj = (jb & 16u) ? t2b : t2a;
              const uint64_t key = ((uint64_t)__float_as_uint(dj) << 32) | (cb + 2 * qp * 16 + jb);
              if (key < top) {
                heap_replace_top(h, KP, key);
                top = h[0];
              }
            }
          }
        }
      }
    }
    // merge the column groups' heaps (group 0 absorbs group 1), then emit
    asm volatile("bar.sync 1, %0;" ::"r"(kThreads - 64));
    if (BF && !row_ok && grp == 0 && active) {
      for (uint32_t i = 0; i < KP; ++i) bf.keys[((uint64_t)blockIdx.x * BM + r) * KP + i] = ~0ull;
    }
    if (row_ok && grp == 0) {
      for (uint32_t g = 1; g < NG; ++g) {
        const uint64_t* o = H + g * BM * KP + r;
        for (uint32_t i = 0; i < KP; ++i) {
          const uint64_t key = o[i * BM];
          if (key < top) {
            heap_replace_top(h, KP, key);
            top = h[0];
          }
        }
      }
      if constexpr (BF) {
        for (uint32_t i = 0; i < KP; ++i) bf.keys[((uint64_t)blockIdx.x * BM + r) * KP + i] = h[i * BM];
      } else {
        for (uint32_t i = 0; i < KP; ++i)
          cand[(uint64_t)prow * KP + i] = h[i * BM] == ~0ull ? kSentinel : (uint32_t)h[i * BM];
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(2 * BN));
  }
}

__global__ void k_mask_norms(const float* norms, const Attr* attr, uint64_t rows, uint64_t padded, float* out) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i < padded) out[i] = (i < rows && attr[i].slot != kNoSlot) ? norms[i] : INFINITY;
}

// hi/lo BF16 split of the phys rows, K padded to a multiple of 64 (zeros)
__global__ void k_split_bf16(const float* X, uint64_t rows, uint32_t dp, uint32_t kp, __nv_bfloat16* hi,
                             __nv_bfloat16* lo) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= rows * kp) return;
  const uint64_t r = i / kp;
  const uint32_t c = (uint32_t)(i % kp);
  const float x = c < dp ? X[r * dp + c] : 0.f;
  const __nv_bfloat16 h = __float2bfloat16_rn(x);
  hi[i] = h;
  lo[i] = __float2bfloat16_rn(x - __bfloat162float(h));
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    GRAB_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p || q != cudaDriverEntryPointSuccess) throw Error(GRAB_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    fn = (EncodeTiledFn)p;
  }
  return fn;
}

static CUtensorMap make_map(void* base, uint64_t rows, uint32_t kp, uint32_t box_rows) {
  CUtensorMap m;
  cuuint64_t dims[2] = {kp, rows};
  cuuint64_t strides[1] = {(cuuint64_t)kp * 2};
  cuuint32_t box[2] = {KCH, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(GRAB_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return m;
}

}  // namespace tc

bool knn_tc_supported(const DevIndex& ix, uint32_t KP) {
  if (getenv("GRAB_KNN_SIMT")) return false;
  (void)ix;  // any d: rows wider than 128 stream A through the ring
  return KP <= tc::KP_MAX;
}

void knn_screen_tc(const DevIndex& ix, const float* norms, const KnnJob* djobs, uint32_t njobs, uint32_t KP,
                   uint32_t* cand, bool causal, cudaStream_t st) {
  using namespace tc;
  const uint32_t kp = (ix.dp + KCH - 1) / KCH * KCH;
  const uint32_t nkc = kp / KCH;
  const uint64_t rows = ix.phys_cap;
  __nv_bfloat16 *hi, *lo;
  GRAB_CUDA(cudaMallocAsync(&hi, rows * kp * 2, st));
  GRAB_CUDA(cudaMallocAsync(&lo, rows * kp * 2, st));
  k_split_bf16<<<(unsigned)div_up(rows * kp, 256), 256, 0, st>>>(ix.X, rows, ix.dp, kp, hi, lo);
  GRAB_CHECK_LAUNCH();
  // candidate |b|^2, +inf for headroom rows and the padding after the last tile
  const uint64_t padded = div_up(rows, BN) * BN + BN;
  float* nm;
  GRAB_CUDA(cudaMallocAsync(&nm, padded * 4, st));
  k_mask_norms<<<(unsigned)div_up(padded, 256), 256, 0, st>>>(norms, ix.attr, rows, padded, nm);
  GRAB_CHECK_LAUNCH();
  const CUtensorMap ahi = make_map(hi, rows, kp, BM), alo = make_map(lo, rows, kp, BM);
  const CUtensorMap bhi = make_map(hi, rows, kp, BN), blo = make_map(lo, rows, kp, BN);
  // prefer two epilogue column groups (8 epilogue warps), then the deepest B ring that fits
  const int stream_a = kp > 128 ? 1 : 0;
  uint32_t stages = 0, ng = 0;
  size_t smem = 0;
  for (uint32_t g = 2; g >= 1 && !stages; --g) {
    for (uint32_t s = MAX_STAGES; s >= 2; --s) {
      const size_t ring = stream_a ? s * 2 * (size_t)(Smem::kChunkA + Smem::kChunkB)
                                   : 2 * (size_t)nkc * BM * 128 + s * 2 * (size_t)nkc * BN * 128;
      const size_t b = 1024 + ring + (size_t)g * BM * KP * 8 + 16 * 8;
      if (b <= 227 * 1024) {
        stages = s;
        ng = g;
        smem = b;
        break;
      }
    }
  }
  if (!stages) throw Error(GRAB_ERR_VALUE, "tensor-core kNN tile exceeds shared memory");
  GRAB_CUDA(cudaFuncSetAttribute(k_knn_screen_tc<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_knn_screen_tc<false><<<njobs, kThreads, smem, st>>>(ahi, alo, bhi, blo, djobs, ix.attr, norms, nm, nkc, KP, cand,
                                                        causal ? 1 : 0, stages, ng, stream_a, TcBf{});
  GRAB_CHECK_LAUNCH();
  GRAB_CUDA(cudaFreeAsync(nm, st));
  GRAB_CUDA(cudaFreeAsync(hi, st));
  GRAB_CUDA(cudaFreeAsync(lo, st));
}

// ring depth / column groups for a screen launch (shared by both modes)
static void tc_config(uint32_t nkc, int stream_a, uint32_t KP, uint32_t& stages, uint32_t& ng, size_t& smem) {
  using namespace tc;
  stages = 0;
  ng = 0;
  for (uint32_t g = 2; g >= 1 && !stages; --g) {
    for (uint32_t s = MAX_STAGES; s >= 2; --s) {
      const size_t ring = stream_a ? s * 2 * (size_t)(Smem::kChunkA + Smem::kChunkB)
                                   : 2 * (size_t)nkc * BM * 128 + s * 2 * (size_t)nkc * BN * 128;
      const size_t b = 1024 + ring + (size_t)g * BM * KP * 8 + 16 * 8;
      if (b <= 227 * 1024) {
        stages = s;
        ng = g;
        smem = b;
        break;
      }
    }
  }
  if (!stages) throw Error(GRAB_ERR_VALUE, "tensor-core kNN tile exceeds shared memory");
}

void bf_screen_tc(const DevIndex& ix, const __nv_bfloat16* q_hi, const __nv_bfloat16* q_lo, const __nv_bfloat16* hi,
                  const __nv_bfloat16* lo, uint32_t ntile, const float* masked_norms, uint32_t KP, TcBf bf,
                  cudaStream_t st) {
  using namespace tc;
  const uint32_t kp = (ix.dp + KCH - 1) / KCH * KCH;
  const uint32_t nkc = kp / KCH;
  const uint64_t rows = ix.phys_cap;
  const uint64_t qrows = (uint64_t)ntile * BM;
  const CUtensorMap ahi = make_map((void*)q_hi, qrows, kp, BM), alo = make_map((void*)q_lo, qrows, kp, BM);
  const CUtensorMap bhi = make_map((void*)hi, rows, kp, BN), blo = make_map((void*)lo, rows, kp, BN);
  const int stream_a = kp > 128 ? 1 : 0;
  uint32_t stages, ng;
  size_t smem;
  tc_config(nkc, stream_a, KP, stages, ng, smem);
  GRAB_CUDA(cudaFuncSetAttribute(k_knn_screen_tc<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_knn_screen_tc<true><<<ntile * bf.S, kThreads, smem, st>>>(ahi, alo, bhi, blo, nullptr, ix.attr, nullptr,
                                                              masked_norms, nkc, KP, nullptr, 0, stages, ng, stream_a,
                                                              bf);
  GRAB_CHECK_LAUNCH();
}

uint32_t tc_pad_cols() { return tc::BN; }

}  // namespace grab
