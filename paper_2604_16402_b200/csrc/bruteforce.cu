// filtered_bruteforce_knn: exact range-filtered top-k by (dist, slot).
// Reference: brute_force_search (evaluate.py:22-44) -- f32 range mask over the
// live rows, f64 distances, stable argsort => (dist, slot) order, short result
// when fewer than k rows qualify.
//
// B200 mapping: the bucket interval [lo, hi] of the range bounds the scan to
// the contiguous slab span [bstart[lo], bstart[hi] + bcount[hi]) -- rows
// outside it cannot satisfy the f32 predicate (bucket_of is monotone), so the
// scan never touches them. One CTA per query, 8 warps striding over the span,
// each warp keeps a sorted top-k list in shared memory; distances use the same
// f64 reduction tree as the search kernel (bit-identical values).
#include "index.cuh"

namespace grab {

struct BfArgs {
  const float* X;
  const Attr* attr;
  uint32_t dp;
  const float* bound;
  uint32_t m;
  const uint32_t* bstart;
  const uint32_t* bcount;
  uint64_t n_live;
  const float* Q;
  const double* lower;
  const double* upper;
  uint64_t range_stride;
  uint32_t k;
  int64_t* out_slots;
  double* out_dists;
  uint32_t* out_counts;
};

constexpr int kBfWarps = 8;
#ifndef GRAB_BF_PF_STEPS
#define GRAB_BF_PF_STEPS 2
#endif

// insert (d, s) into the sorted warp list (length k, +inf padded) if it beats the tail
__device__ __forceinline__ void list_insert(double* ld, uint32_t* ls, uint32_t k, double d, uint32_t s) {
  const uint32_t lane = lane_id();
  if (!key_less(d, s, ld[k - 1], ls[k - 1])) return;  // warp-uniform
  uint32_t pos = 0;
  for (uint32_t b0 = 0; b0 < k; b0 += 32) {
    uint32_t i = b0 + lane;
    bool lt = i < k && key_less(ld[i], ls[i], d, s);
    pos += __popc(__ballot_sync(0xFFFFFFFFu, lt));
  }
  // shift [pos, k-1) right by one, from the tail backwards in 32-wide chunks
  for (int32_t hi = (int32_t)k - 1; hi > (int32_t)pos; hi -= 32) {
    int32_t i = hi - (int32_t)lane;
    double dv = 0;
    uint32_t sv = 0;
    bool mv = i > (int32_t)pos;
    if (mv) {
      dv = ld[i - 1];
      sv = ls[i - 1];
    }
    __syncwarp();
    if (mv) {
      ld[i] = dv;
      ls[i] = sv;
    }
    __syncwarp();
  }
  __syncwarp();  // every lane has read the list (no shift ran when pos == k - 1)
  if (lane == 0) {
    ld[pos] = d;
    ls[pos] = s;
  }
  __syncwarp();
}

template <int NC>
__global__ void __launch_bounds__(kBfWarps * 32) k_bruteforce(BfArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  const uint32_t lane = lane_id(), wid = threadIdx.x >> 5;
  const uint32_t k = a.k;
  double* ld = (double*)smem + (uint64_t)wid * k;
  uint32_t* ls = (uint32_t*)((double*)smem + (uint64_t)kBfWarps * k) + (uint64_t)wid * k;
  const uint64_t qi = blockIdx.x;
  for (uint32_t i = lane; i < k; i += 32) {
    ld[i] = __longlong_as_double(0x7FF0000000000000ll);
    ls[i] = kNoSlot;
  }
  __syncwarp();
  const float lo_f = __double2float_rn(a.lower[qi * a.range_stride]);
  const float hi_f = __double2float_rn(a.upper[qi * a.range_stride]);
  float4 q[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    uint32_t col = (c * 32 + lane) * 4;
    q[c] = col < a.dp ? *reinterpret_cast<const float4*>(a.Q + qi * a.dp + col) : make_float4(0, 0, 0, 0);
  }
  // !(lo <= hi) (inverted or NaN bounds on the device path): empty result, never a
  // wrapped bucket interval
  if (a.m > 0 && a.n_live > 0 && lo_f <= hi_f) {
    const uint32_t lo_b = bucket_of_f32(a.bound, a.m, lo_f), hi_b = bucket_of_f32(a.bound, a.m, hi_f);
    const uint32_t p0 = __ldg(a.bstart + lo_b), p1 = __ldg(a.bstart + hi_b) + __ldg(a.bcount + hi_b);
    constexpr int G = NC == 1 ? 8 : (NC == 2 ? 4 : (NC <= 4 ? 2 : 1));
    const uint32_t rowb = a.dp * 4;
    for (uint32_t base = p0 + wid * G; base < p1; base += kBfWarps * G) {
      // G consecutive rows per warp step; the warp's rows two steps ahead are
      // one contiguous block: a single bulk L2 prefetch covers them
      {
        const uint32_t pf = base + GRAB_BF_PF_STEPS * kBfWarps * G;
        if (lane == 0 && pf + G <= p1)
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.X + (uint64_t)pf * a.dp),
                       "r"(rowb * (uint32_t)G)
                       : "memory");
      }
      bool ok[G];
      uint32_t slot[G];
      float4 x[G][NC];
      // the row loads do not wait for the attribute test (every row of the span
      // is mapped; rows that fail it are dropped after the reduction)
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const uint32_t p = base + g;
        const uint32_t pc = p < p1 ? p : p0;
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          uint32_t col = (c * 32 + lane) * 4;
          x[g][c] = col < a.dp ? ldg_nc_f4(a.X + (uint64_t)pc * a.dp + col) : make_float4(0, 0, 0, 0);
        }
        ok[g] = false;
        slot[g] = kNoSlot;
        if (p < p1) {
          Attr at = ld_attr(a.attr, p);
          slot[g] = at.slot;
          ok[g] = at.slot < a.n_live && at.s >= lo_f && at.s <= hi_f;
        }
      }
      double part[G];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        double acc = 0.0;
#pragma unroll
        for (int c = 0; c < NC; ++c) acc = sq4(x[g][c], q[c], acc);
        part[g] = acc;
      }
      // one scatter-reduction for the G rows (same pairing tree as warp_sum:
      // bit-identical), row g's sum on lane g << SH
      const double sum = reduce_scatter<G>(part);
      constexpr uint32_t SH = G == 8 ? 2 : (G == 4 ? 3 : (G == 2 ? 4 : 5));
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const double dg = __shfl_sync(0xFFFFFFFFu, sum, (uint32_t)g << SH);
        if (!ok[g]) continue;  // uniform: same row for all lanes
        list_insert(ld, ls, k, dg, slot[g]);
      }
    }
  }
  __syncthreads();
  if (wid == 0) {
    for (uint32_t w = 1; w < kBfWarps; ++w) {
      double* od = (double*)smem + (uint64_t)w * k;
      uint32_t* os = (uint32_t*)((double*)smem + (uint64_t)kBfWarps * k) + (uint64_t)w * k;
      for (uint32_t i = 0; i < k; ++i) {
        double d = od[i];
        uint32_t s = os[i];
        if (s == kNoSlot) break;
        list_insert(ld, ls, k, d, s);
      }
    }
    uint32_t cnt = 0;
    for (uint32_t b0 = 0; b0 < k; b0 += 32) {
      uint32_t i = b0 + lane;
      bool v = i < k && ls[i] != kNoSlot;
      cnt += __popc(__ballot_sync(0xFFFFFFFFu, v));
      if (i < k) {
        a.out_slots[qi * k + i] = v ? (int64_t)ls[i] : -1;
        a.out_dists[qi * k + i] = v ? ld[i] : __longlong_as_double(0x7FF8000000000000ll);
      }
    }
    if (lane == 0) a.out_counts[qi] = cnt;
  }
}

void run_bruteforce(const DevIndex& ix, const float* Q, uint64_t nq, const double* lo, const double* hi,
                    uint64_t stride, uint32_t k, uint64_t n_live, int64_t* os, double* od, uint32_t* oc,
                    cudaStream_t st) {
  if (!nq) return;
  BfArgs a{ix.X, ix.attr, ix.dp, ix.bound, ix.m, ix.bstart, ix.bcount, n_live, Q, lo, hi, stride, k, os, od, oc};
  size_t smem = (size_t)kBfWarps * k * 12;
  if (smem > 200 * 1024) throw Error(GRAB_ERR_VALUE, "brute force k too large");
  uint32_t nc = (uint32_t)div_up(ix.dp, 128);
  auto go = [&](auto kern) {
    GRAB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<(unsigned)nq, kBfWarps * 32, smem, st>>>(a);
    GRAB_CHECK_LAUNCH();
  };
  if (nc <= 1)
    go(k_bruteforce<1>);
  else if (nc <= 2)
    go(k_bruteforce<2>);
  else if (nc <= 4)
    go(k_bruteforce<4>);
  else if (nc <= 8)
    go(k_bruteforce<8>);
  else if (nc <= 16)
    go(k_bruteforce<16>);
  else
    throw Error(GRAB_ERR_VALUE, "dimension > 2048 not supported");
}

}  // namespace grab

namespace grab {

// sq_distances (core.py:25-38): one warp per row, the library's f64 tree.
template <int NC>
__global__ void k_sq_distances(const float* q, const float* rows, uint64_t n, uint32_t dp, double* out) {
  const uint64_t r = blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= n) return;
  const uint32_t lane = lane_id();
  double acc = 0.0;
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    uint32_t col = (c * 32 + lane) * 4;
    if (col < dp)
      acc = sq4(*reinterpret_cast<const float4*>(rows + r * dp + col), *reinterpret_cast<const float4*>(q + col), acc);
  }
  acc = warp_sum(acc);
  if (lane == 0) out[r] = acc;
}

void run_sq_distances(const float* q, const float* rows, uint64_t n, uint32_t dp, double* out, cudaStream_t st) {
  unsigned blocks = (unsigned)div_up(n, 4);
  uint32_t nc = (uint32_t)div_up(dp, 128);
  if (nc <= 1)
    k_sq_distances<1><<<blocks, 128, 0, st>>>(q, rows, n, dp, out);
  else if (nc <= 2)
    k_sq_distances<2><<<blocks, 128, 0, st>>>(q, rows, n, dp, out);
  else if (nc <= 4)
    k_sq_distances<4><<<blocks, 128, 0, st>>>(q, rows, n, dp, out);
  else if (nc <= 8)
    k_sq_distances<8><<<blocks, 128, 0, st>>>(q, rows, n, dp, out);
  else if (nc <= 16)
    k_sq_distances<16><<<blocks, 128, 0, st>>>(q, rows, n, dp, out);
  else
    throw Error(GRAB_ERR_VALUE, "dimension > 2048 not supported");
  GRAB_CHECK_LAUNCH();
}

}  // namespace grab
