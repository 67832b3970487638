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
#include <cstdio>
#include <cstdlib>

#include <cub/cub.cuh>

#include "index.cuh"
#include "knn.cuh"

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

// qmap / nmap (optional): block b handles query qmap[b] when b < *nmap (the
// tensor-core path's fallback list), else nothing
template <int NC>
__global__ void __launch_bounds__(kBfWarps * 32) k_bruteforce(BfArgs a, const uint32_t* qmap, const uint32_t* nmap) {
  extern __shared__ __align__(16) uint8_t smem[];
  const uint32_t lane = lane_id(), wid = threadIdx.x >> 5;
  const uint32_t k = a.k;
  double* ld = (double*)smem + (uint64_t)wid * k;
  uint32_t* ls = (uint32_t*)((double*)smem + (uint64_t)kBfWarps * k) + (uint64_t)wid * k;
  if (qmap && blockIdx.x >= *nmap) return;
  const uint64_t qi = qmap ? qmap[blockIdx.x] : blockIdx.x;
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

static void run_bruteforce_simt(const BfArgs& a, uint32_t dp, uint64_t nq, const uint32_t* qmap,
                                const uint32_t* nmap, cudaStream_t st) {
  const uint32_t k = a.k;
  size_t smem = (size_t)kBfWarps * k * 12;
  if (smem > 200 * 1024) throw Error(GRAB_ERR_VALUE, "brute force k too large");
  uint32_t nc = (uint32_t)div_up(dp, 128);
  auto go = [&](auto kern) {
    GRAB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<(unsigned)nq, kBfWarps * 32, smem, st>>>(a, qmap, nmap);
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

// ---------------------------------------------------------------- tensor-core path
// Batched brute force on the tcgen05 screen (knn_tc.cu, BF mode):
//   1. k_bf_prep      per query: f32 bounds -> bucket interval -> slab span [p0, p1)
//   2. radix sort     queries by p0, so a tile of 128 sorted queries has nearly one span
//   3. k_bf_gather    sorted query rows split hi/lo BF16 (the screen's A operand),
//                     |q|^2, bounds; per tile the union span (atomic min / max)
//   4. bf_screen_tc   split-BF16 UMMA over the tile's span, S CTAs per tile, each
//                     keeping every row's KP = k + 16 smallest screen distances
//                     among in-range live columns (a heap per row and split)
//   5. k_bf_rerank    per query: exact f64 distances (the library's one reduction
//                     tree: bit-identical to the SIMT scan) of the candidates that
//                     can still be in the top k, top-k by (dist, slot), and a
//                     completeness proof: every column a heap dropped has screen
//                     distance >= its heap's kept maximum T_s, and the screen is
//                     within err = 2^-12 (|q|^2 + max |x|^2) of the exact value,
//                     so T_s - err > (exact k-th) shows nothing was missed
//   6. k_bruteforce   (SIMT) re-runs exactly the queries whose proof failed
// Screen error bound: x = hi + lo + r, |r| <= 2^-17 |x|; the dropped lo*lo and
// residual terms plus fp32 accumulation over 3 * d products stay below
// 5e-5 (|q|^2 + |x|^2) at d <= 2048 (derivation in DESIGN.md); 2^-12 leaves 4x.
constexpr uint32_t kBfTcMargin = 16;
constexpr uint32_t kBfTcBM = 128;

__global__ void k_bf_prep(BfArgs a, uint64_t nq, uint32_t* key, uint32_t* idx, uint32_t* p0s, uint32_t* p1s) {
  const uint64_t qi = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (qi >= nq) return;
  const float lo_f = __double2float_rn(a.lower[qi * a.range_stride]);
  const float hi_f = __double2float_rn(a.upper[qi * a.range_stride]);
  uint32_t p0 = 0, p1 = 0;
  if (a.m > 0 && a.n_live > 0 && lo_f <= hi_f) {
    const uint32_t lo_b = bucket_of_f32(a.bound, a.m, lo_f), hi_b = bucket_of_f32(a.bound, a.m, hi_f);
    p0 = __ldg(a.bstart + lo_b);
    p1 = __ldg(a.bstart + hi_b) + __ldg(a.bcount + hi_b);
  }
  key[qi] = p0;
  idx[qi] = (uint32_t)qi;
  p0s[qi] = p0;
  p1s[qi] = p1;
}

// warp per sorted row rs < ntile * 128
__global__ void k_bf_gather(BfArgs a, uint64_t nq, uint64_t nrows, uint32_t kp, const uint32_t* perm,
                            const uint32_t* p0s, const uint32_t* p1s, __nv_bfloat16* qh, __nv_bfloat16* ql,
                            float* qnorm, float* qlo, float* qhi, uint32_t* span) {
  const uint64_t rs = blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (rs >= nrows) return;
  const uint32_t lane = lane_id();
  bool valid = false;
  uint32_t qi = 0, p0 = 0, p1 = 0;
  if (rs < nq) {
    qi = perm[rs];
    p0 = p0s[qi];
    p1 = p1s[qi];
    valid = p1 > p0;
  }
  float acc = 0.f;
  for (uint32_t c = lane; c < kp; c += 32) {
    const float x = (valid && c < a.dp) ? a.Q[(uint64_t)qi * a.dp + c] : 0.f;
    const __nv_bfloat16 h = __float2bfloat16_rn(x);  // knn_tc.cu k_split_bf16's split
    qh[rs * kp + c] = h;
    ql[rs * kp + c] = __float2bfloat16_rn(x - __bfloat162float(h));
    acc = fmaf(x, x, acc);
  }
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, o);
  if (lane == 0) {
    qnorm[rs] = acc;
    qlo[rs] = valid ? __double2float_rn(a.lower[qi * a.range_stride]) : INFINITY;
    qhi[rs] = valid ? __double2float_rn(a.upper[qi * a.range_stride]) : -INFINITY;
    if (valid) {
      atomicMin(span + 2 * (rs / kBfTcBM), p0);
      atomicMax(span + 2 * (rs / kBfTcBM) + 1, p1);
    }
  }
}

__global__ void k_bf_span_init(uint32_t* span, uint32_t ntile) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < ntile) {
    span[2 * t] = 0xFFFFFFFFu;
    span[2 * t + 1] = 0u;
  }
}

// One pass over X for the screen's B operand: the hi/lo BF16 split of every
// phys row (knn_tc.cu k_split_bf16's rounding, K padded to kp with zeros), its
// |x|^2 (+inf when the row is not live) and the max live |x|^2. Warp per row,
// float4 per lane (16-byte loads, 8-byte stores).
__global__ void __launch_bounds__(256) k_bf_xprep(const float* __restrict__ X, const Attr* __restrict__ attr,
                                                  uint64_t rows, uint64_t padded, uint32_t dp, uint32_t kp,
                                                  uint64_t n_live, __nv_bfloat16* __restrict__ xh,
                                                  __nv_bfloat16* __restrict__ xl, float* __restrict__ nm,
                                                  uint32_t* maxn) {
  __shared__ float wmax[8];
  const uint64_t r = blockIdx.x * 8ull + (threadIdx.x >> 5);
  const uint32_t lane = lane_id();
  float acc = 0.f;
  bool live = false;
  if (r < rows) {
    live = attr[r].slot < n_live;
    for (uint32_t c = lane * 4; c < kp; c += 128) {
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (c < dp) v = *reinterpret_cast<const float4*>(X + r * dp + c);
      const float f[4] = {v.x, v.y, v.z, v.w};
      __nv_bfloat16 h[4], l[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        h[j] = __float2bfloat16_rn(f[j]);
        l[j] = __float2bfloat16_rn(f[j] - __bfloat162float(h[j]));
        acc = fmaf(f[j], f[j], acc);
      }
      *reinterpret_cast<uint2*>(xh + r * kp + c) = *reinterpret_cast<const uint2*>(h);
      *reinterpret_cast<uint2*>(xl + r * kp + c) = *reinterpret_cast<const uint2*>(l);
    }
  }
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, o);
  if (lane == 0) {
    if (r < padded) nm[r] = live ? acc : INFINITY;
    wmax[threadIdx.x >> 5] = live ? acc : 0.f;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float mx = 0.f;
    for (int w = 0; w < 8; ++w) mx = fmaxf(mx, wmax[w]);
    if (mx > 0.f) atomicMax(maxn, __float_as_uint(mx));  // non-negative floats order as their bits
  }
}

// Warp per sorted query row. smem per warp: S*KP keys + k (dist, slot) list + the rerank list.
template <int NC>
__global__ void __launch_bounds__(128) k_bf_rerank(BfArgs a, uint64_t nq, const uint32_t* perm, const uint64_t* keys,
                                                   uint32_t S, uint32_t KP, const float* qnorm, const float* qlo,
                                                   const float* qhi, const uint32_t* maxn, uint32_t* fb_list,
                                                   uint32_t* fb_count) {
  extern __shared__ __align__(16) uint8_t smem[];
  const uint32_t lane = lane_id(), wib = threadIdx.x >> 5;
  const uint64_t rs = blockIdx.x * 4ull + wib;
  if (rs >= nq) return;
  const uint32_t k = a.k, n = S * KP;
  const size_t per_warp = (size_t)n * 8 + (size_t)k * 12 + (size_t)n * 4;
  uint8_t* base = smem + (size_t)wib * ((per_warp + 15) & ~(size_t)15);
  uint64_t* kk = (uint64_t*)base;
  double* ld = (double*)(base + (size_t)n * 8);
  uint32_t* ls = (uint32_t*)(ld + k);
  uint32_t* rl = ls + k;  // rerank list (phys)
  const uint32_t qi = perm[rs];
  const uint32_t tile = (uint32_t)(rs / kBfTcBM), r = (uint32_t)(rs % kBfTcBM);
  for (uint32_t i = lane; i < k; i += 32) {
    ld[i] = __longlong_as_double(0x7FF0000000000000ll);
    ls[i] = kNoSlot;
  }
  uint32_t cnt = 0;
  bool fail = false;
  if (qlo[rs] <= qhi[rs]) {
    uint32_t nvalid = 0;
    for (uint32_t i = lane; i < n; i += 32) {
      const uint32_t s = i / KP, j = i - s * KP;
      const uint64_t key = keys[(((uint64_t)tile * S + s) * kBfTcBM + r) * KP + j];
      kk[i] = key;
      nvalid += key != ~0ull;
    }
    for (int o = 16; o; o >>= 1) nvalid += __shfl_xor_sync(0xFFFFFFFFu, nvalid, o);
    __syncwarp();
    // k-th smallest screen distance (f32 bits of non-negative floats order as u32)
    uint32_t dk = 0x7F800000u;
    if (nvalid >= k) {
      uint32_t lo = 0, hi = 0x7F800000u;  // smallest v with #(bits <= v) >= k
      while (lo < hi) {
        const uint32_t mid = lo + ((hi - lo) >> 1);
        uint32_t c = 0;
        for (uint32_t i = lane; i < n; i += 32) {
          const uint64_t key = kk[i];
          c += key != ~0ull && (uint32_t)(key >> 32) <= mid;
        }
        for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xFFFFFFFFu, c, o);
        if (c >= k)
          hi = mid;
        else
          lo = mid + 1;
      }
      dk = lo;
    }
    const double err = ldexp((double)qnorm[rs] + (double)__uint_as_float(*maxn), -12);
    const double thr = (double)__uint_as_float(dk) + 2.0 * err;
    // candidates that can still be in the top k, in list order
    uint32_t nr = 0;
    for (uint32_t b0 = 0; b0 < n; b0 += 32) {
      const uint32_t i = b0 + lane;
      uint64_t key = ~0ull;
      if (i < n) key = kk[i];
      const bool take = key != ~0ull && (double)__uint_as_float((uint32_t)(key >> 32)) <= thr;
      const uint32_t m = __ballot_sync(0xFFFFFFFFu, take);
      if (take) rl[nr + __popc(m & ((1u << lane) - 1))] = (uint32_t)key;
      nr += __popc(m);
    }
    __syncwarp();
    // exact f64 distances (warp_sum: the tree every kernel uses) + (dist, slot) top-k
    float4 q[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const uint32_t col = (c * 32 + lane) * 4;
      q[c] = col < a.dp ? *reinterpret_cast<const float4*>(a.Q + (uint64_t)qi * a.dp + col)
                        : make_float4(0, 0, 0, 0);
    }
    for (uint32_t i = 0; i < nr; ++i) {
      const uint32_t p = rl[i];
      double acc = 0.0;
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const uint32_t col = (c * 32 + lane) * 4;
        const float4 x = col < a.dp ? ldg_nc_f4(a.X + (uint64_t)p * a.dp + col) : make_float4(0, 0, 0, 0);
        acc = sq4(x, q[c], acc);
      }
      acc = warp_sum(acc);
      list_insert(ld, ls, k, acc, __ldg(&a.attr[p].slot));
    }
    for (uint32_t b0 = 0; b0 < k; b0 += 32) cnt += __popc(__ballot_sync(0xFFFFFFFFu, b0 + lane < k && ls[b0 + lane] != kNoSlot));
    // completeness: a full heap (root != ~0) dropped only columns with screen
    // distance >= its root; those are exactly farther than the k-th when
    // root - err > exact k-th (a short result needs every heap non-full)
    const double dstar = cnt >= k ? ld[k - 1] : __longlong_as_double(0x7FF0000000000000ll);
    bool bad = false;
    for (uint32_t s = lane; s < S; s += 32) {
      const uint64_t root = kk[s * KP];
      if (root != ~0ull) bad |= !((double)__uint_as_float((uint32_t)(root >> 32)) - err > dstar);
    }
    fail = __any_sync(0xFFFFFFFFu, bad);
  }
  if (fail) {
    if (lane == 0) fb_list[atomicAdd(fb_count, 1u)] = qi;
    return;
  }
  for (uint32_t i = lane; i < k; i += 32) {
    const bool v = i < cnt;
    a.out_slots[(uint64_t)qi * k + i] = v ? (int64_t)ls[i] : -1;
    a.out_dists[(uint64_t)qi * k + i] = v ? ld[i] : __longlong_as_double(0x7FF8000000000000ll);
  }
  if (lane == 0) a.out_counts[qi] = cnt;
}

static bool bf_tc_enabled(const DevIndex& ix, uint32_t k, uint64_t nq) {
  if (getenv("GRAB_BF_SIMT")) return false;
  return ix.m > 0 && nq >= 64 && k + kBfTcMargin <= 80 && ix.phys_cap < 0x7FFFFFFFull;
}

void run_bruteforce(const DevIndex& ix, const float* Q, uint64_t nq, const double* lo, const double* hi,
                    uint64_t stride, uint32_t k, uint64_t n_live, int64_t* os, double* od, uint32_t* oc,
                    cudaStream_t st) {
  if (!nq) return;
  BfArgs a{ix.X, ix.attr, ix.dp, ix.bound, ix.m, ix.bstart, ix.bcount, n_live, Q, lo, hi, stride, k, os, od, oc};
  if (!bf_tc_enabled(ix, k, nq)) {
    run_bruteforce_simt(a, ix.dp, nq, nullptr, nullptr, st);
    return;
  }
  const uint32_t KP = (k + kBfTcMargin + 7) / 8 * 8;
  const uint32_t kp = (ix.dp + 63) / 64 * 64;
  const uint32_t ntile = (uint32_t)div_up(nq, kBfTcBM);
  const uint64_t nrows = (uint64_t)ntile * kBfTcBM;
  // splits per tile: ~4 CTAs per SM over the whole launch, at most 32
  const uint32_t S = (uint32_t)std::min<uint64_t>(32, std::max<uint64_t>(1, div_up(4ull * ix.num_sms, ntile)));
  const uint64_t padded = div_up(ix.phys_cap, tc_pad_cols()) * tc_pad_cols() + tc_pad_cols();
  // one scratch allocation (stream-ordered pool)
  size_t off = 0;
  auto carve = [&](size_t bytes) {
    const size_t o = off;
    off += (bytes + 255) & ~(size_t)255;
    return o;
  };
  const size_t o_key = carve(nq * 4), o_idx = carve(nq * 4), o_skey = carve(nq * 4), o_perm = carve(nq * 4);
  const size_t o_p0 = carve(nq * 4), o_p1 = carve(nq * 4), o_qh = carve(nrows * kp * 2), o_ql = carve(nrows * kp * 2);
  const size_t o_qn = carve(nrows * 4), o_qlo = carve(nrows * 4), o_qhi = carve(nrows * 4);
  const size_t o_span = carve((size_t)ntile * 8), o_nm = carve(padded * 4), o_maxn = carve(16);
  const size_t o_keys = carve((size_t)ntile * S * kBfTcBM * KP * 8), o_fb = carve(nq * 4);
  size_t sort_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, (uint32_t*)nullptr, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (uint32_t*)nullptr, (int)nq, 0, 32, st);
  const size_t o_sort = carve(sort_bytes);
  uint8_t* w;
  GRAB_CUDA(cudaMallocAsync(&w, off, st));
  auto U = [&](size_t o) { return (uint32_t*)(w + o); };
  k_bf_prep<<<(unsigned)div_up(nq, 256), 256, 0, st>>>(a, nq, U(o_key), U(o_idx), U(o_p0), U(o_p1));
  GRAB_CHECK_LAUNCH();
  GRAB_CUDA(cub::DeviceRadixSort::SortPairs(w + o_sort, sort_bytes, U(o_key), U(o_skey), U(o_idx), U(o_perm), (int)nq,
                                            0, 32, st));
  k_bf_span_init<<<(unsigned)div_up(ntile, 128), 128, 0, st>>>(U(o_span), ntile);
  GRAB_CHECK_LAUNCH();
  __nv_bfloat16* qh = (__nv_bfloat16*)(w + o_qh);
  __nv_bfloat16* ql = (__nv_bfloat16*)(w + o_ql);
  float* qn = (float*)(w + o_qn);
  float* qlo = (float*)(w + o_qlo);
  float* qhi = (float*)(w + o_qhi);
  k_bf_gather<<<(unsigned)div_up(nrows, 8), 256, 0, st>>>(a, nq, nrows, kp, U(o_perm), U(o_p0), U(o_p1), qh, ql, qn,
                                                          qlo, qhi, U(o_span));
  GRAB_CHECK_LAUNCH();
  GRAB_CUDA(cudaMemsetAsync(w + o_maxn, 0, 16, st));
  float* nm = (float*)(w + o_nm);
  __nv_bfloat16 *xh, *xl;
  GRAB_CUDA(cudaMallocAsync(&xh, ix.phys_cap * kp * 2, st));
  GRAB_CUDA(cudaMallocAsync(&xl, ix.phys_cap * kp * 2, st));
  k_bf_xprep<<<(unsigned)div_up(padded, 8), 256, 0, st>>>(ix.X, ix.attr, ix.phys_cap, padded, ix.dp, kp, n_live, xh,
                                                          xl, nm, U(o_maxn));
  GRAB_CHECK_LAUNCH();
  TcBf bf;
  bf.qnorm = qn;
  bf.qlo = qlo;
  bf.qhi = qhi;
  bf.span = U(o_span);
  bf.S = S;
  bf.keys = (uint64_t*)(w + o_keys);
  bf_screen_tc(ix, qh, ql, xh, xl, ntile, nm, KP, bf, st);
  GRAB_CUDA(cudaFreeAsync(xh, st));
  GRAB_CUDA(cudaFreeAsync(xl, st));
  uint32_t* fb_count = U(o_maxn) + 1;
  const size_t per_warp = ((size_t)S * KP * 12 + (size_t)k * 12 + 15) & ~(size_t)15;
  const size_t rsmem = 4 * per_warp;
  if (rsmem > 200 * 1024) throw Error(GRAB_ERR_VALUE, "brute force k too large");
  uint32_t nc = (uint32_t)div_up(ix.dp, 128);
  auto rr = [&](auto kern) {
    GRAB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsmem));
    kern<<<(unsigned)div_up(nq, 4), 128, rsmem, st>>>(a, nq, U(o_perm), bf.keys, S, KP, qn, qlo, qhi, U(o_maxn),
                                                      U(o_fb), fb_count);
    GRAB_CHECK_LAUNCH();
  };
  if (nc <= 1)
    rr(k_bf_rerank<1>);
  else if (nc <= 2)
    rr(k_bf_rerank<2>);
  else if (nc <= 4)
    rr(k_bf_rerank<4>);
  else if (nc <= 8)
    rr(k_bf_rerank<8>);
  else if (nc <= 16)
    rr(k_bf_rerank<16>);
  else
    throw Error(GRAB_ERR_VALUE, "dimension > 2048 not supported");
  // exact re-run of the queries whose completeness proof failed (normally none)
  run_bruteforce_simt(a, ix.dp, nq, U(o_fb), fb_count, st);
  if (getenv("GRAB_BF_DEBUG")) {  // (test / lab hook: synchronises)
    uint32_t nfb = 0;
    GRAB_CUDA(cudaMemcpyAsync(&nfb, fb_count, 4, cudaMemcpyDeviceToHost, st));
    GRAB_CUDA(cudaStreamSynchronize(st));
    fprintf(stderr, "[grab] brute force tc: %llu queries, %u tiles x %u splits, KP %u, simt re-runs %u\n",
            (unsigned long long)nq, ntile, S, KP, nfb);
  }
  GRAB_CUDA(cudaFreeAsync(w, st));
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
