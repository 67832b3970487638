// Append-only batched insertion (reference updater.py:154-263).
//
//   append            append_batch (layout.py:181-223): tail claim, bucket ids,
//                     zero-shift slab placement (relayout only on slab overflow)
//   candidates        _bucket_candidates (updater.py:126-151): exact in-bucket
//                     top-2*K_max among members with slot < q (causal kNN on the
//                     slab), plus a full-range beam search (itopk = k = 128,
//                     width 4, 50 iterations, live_count = n0, seed =
//                     derive_query_seed(rng_seed, q)) for every fresh q at once
//   forward           union, (dist, slot) order, nearest pre-batch node,
//                     select_neighbors (updater.py:49-84), intra-then-cross row
//   reverse           requests sorted by (v, q); one warp per target v applies
//                     try_rewire (updater.py:87-123) serially, targets in parallel
//   heal              _heal_unreachable (updater.py:266-324), sequential warp
//
// The forward stage only reads rows < n0 and writes fresh rows, so it runs for
// the whole batch in parallel without changing the result.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_select.cuh>
#include <cub/iterator/counting_input_iterator.cuh>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <vector>

#include "index.cuh"
#include "knn.cuh"
#include "ops.cuh"
#include "search.cuh"

namespace grab {

static double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

struct Pool {
  std::vector<void*> ptrs;
  cudaStream_t st;
  explicit Pool(cudaStream_t s) : st(s) {}
  template <class T>
  T* alloc(size_t n) {
    void* p = nullptr;
    GRAB_CUDA(cudaMallocAsync(&p, std::max<size_t>(n, 1) * sizeof(T), st));
    ptrs.push_back(p);
    return (T*)p;
  }
  ~Pool() {
    for (void* p : ptrs) cudaFreeAsync(p, st);
  }
};

// ------------------------------------------------------------- warp distance
template <int NC>
struct RowRegs {
  float4 v[NC];
};

template <int NC>
__device__ __forceinline__ void load_row(RowRegs<NC>& r, const float* X, uint32_t dp, uint32_t p) {
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    uint32_t col = (c * 32 + lane_id()) * 4;
    r.v[c] = col < dp ? *reinterpret_cast<const float4*>(X + (uint64_t)p * dp + col) : make_float4(0, 0, 0, 0);
  }
}

template <int NC>
__device__ __forceinline__ double row_dist(const RowRegs<NC>& q, const float* X, uint32_t dp, uint32_t p) {
  double acc = 0.0;
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    uint32_t col = (c * 32 + lane_id()) * 4;
    if (col < dp) acc = sq4(ldg_nc_f4(X + (uint64_t)p * dp + col), q.v[c], acc);
  }
  return warp_sum(acc);
}

// G candidate rows in flight per round (x: G * NC float4 registers); the
// distance of row g lands on lanes with lane >> SH == g.
template <int NC>
struct Batch {
  static constexpr int G = NC == 1 ? 8 : (NC == 2 ? 4 : (NC <= 8 ? 2 : 1));
  static constexpr int SH = G == 8 ? 2 : (G == 4 ? 3 : (G == 2 ? 4 : 5));
};

// Distances from `r` to rows p[0..G) (ok[g] false: row not read, partial 0);
// same per-lane chain and reduction tree as row_dist, so bit-identical to it.
template <int NC>
__device__ __forceinline__ double dist_batch(const RowRegs<NC>& r, const float* X, uint32_t dp,
                                             const uint32_t (&p)[Batch<NC>::G], const bool (&ok)[Batch<NC>::G]) {
  constexpr int G = Batch<NC>::G;
  const uint32_t lane = lane_id();
  float4 x[G][NC];
#pragma unroll
  for (int g = 0; g < G; ++g)
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const uint32_t col = (c * 32 + lane) * 4;
      x[g][c] = (ok[g] && col < dp) ? ldg_nc_f4(X + (uint64_t)p[g] * dp + col) : make_float4(0, 0, 0, 0);
    }
  double part[G];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    double acc = 0.0;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const uint32_t col = (c * 32 + lane) * 4;
      if (col < dp) acc = sq4(x[g][c], r.v[c], acc);
    }
    part[g] = acc;
  }
  return reduce_scatter<G>(part);
}

// f32 screen of the same G rows: direct differences, one FMA chain per lane and
// the same pairing tree in f32. Within kScreenRel * value of the exact (f64)
// distance: <= (dp / 32 + 8) roundings of 2^-24 relative each, all terms >= 0.
template <int G>
__device__ __forceinline__ float reduce_scatter_f32(float (&p)[G]) {
  const uint32_t lane = threadIdx.x & 31u;
  if constexpr (G == 1) {
    float t = p[0];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xFFFFFFFFu, t, o);
    return t;
  } else {
    constexpr int H = G / 2;
    float q[H];
    const bool hi = (lane & 16u) != 0;
#pragma unroll
    for (int j = 0; j < H; ++j) {
      const float send = hi ? p[j] : p[H + j];
      const float keep = hi ? p[H + j] : p[j];
      q[j] = keep + __shfl_xor_sync(0xFFFFFFFFu, send, 16);
    }
    if constexpr (H == 1) {
      float t = q[0];
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) t += __shfl_xor_sync(0xFFFFFFFFu, t, o);
      return t;
    } else {
      constexpr int H2 = H / 2;
      float r[H2];
      const bool hi2 = (lane & 8u) != 0;
#pragma unroll
      for (int j = 0; j < H2; ++j) {
        const float send = hi2 ? q[j] : q[H2 + j];
        const float keep = hi2 ? q[H2 + j] : q[j];
        r[j] = keep + __shfl_xor_sync(0xFFFFFFFFu, send, 8);
      }
      if constexpr (H2 == 1) {
        float t = r[0];
#pragma unroll
        for (int o = 4; o > 0; o >>= 1) t += __shfl_xor_sync(0xFFFFFFFFu, t, o);
        return t;
      } else {
        const bool hi3 = (lane & 4u) != 0;
        const float send = hi3 ? r[0] : r[1];
        const float keep = hi3 ? r[1] : r[0];
        float t = keep + __shfl_xor_sync(0xFFFFFFFFu, send, 4);
        t += __shfl_xor_sync(0xFFFFFFFFu, t, 2);
        t += __shfl_xor_sync(0xFFFFFFFFu, t, 1);
        return t;
      }
    }
  }
}

template <int NC>
__device__ __forceinline__ float dist_batch_f32(const RowRegs<NC>& r, const float* X, uint32_t dp,
                                                const uint32_t (&p)[Batch<NC>::G], const bool (&ok)[Batch<NC>::G]) {
  constexpr int G = Batch<NC>::G;
  const uint32_t lane = lane_id();
  float4 x[G][NC];
#pragma unroll
  for (int g = 0; g < G; ++g)
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const uint32_t col = (c * 32 + lane) * 4;
      x[g][c] = (ok[g] && col < dp) ? ldg_nc_f4(X + (uint64_t)p[g] * dp + col) : make_float4(0, 0, 0, 0);
    }
  float part[G];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    float acc = 0.f;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const uint32_t col = (c * 32 + lane) * 4;
      if (col < dp) {
        const float4 q = r.v[c];
        float d = x[g][c].x - q.x;
        acc = fmaf(d, d, acc);
        d = x[g][c].y - q.y;
        acc = fmaf(d, d, acc);
        d = x[g][c].z - q.z;
        acc = fmaf(d, d, acc);
        d = x[g][c].w - q.w;
        acc = fmaf(d, d, acc);
      }
    }
    part[g] = acc;
  }
  return reduce_scatter_f32<G>(part);
}

// relative error bound of the f32 screen for rows of dp floats (generous: 4x)
__device__ __forceinline__ double screen_rel(uint32_t dp) {
  return fmax(ldexp(1.0, -16), (double)(dp / 32 + 8) * ldexp(1.0, -22));
}

// ------------------------------------------------------------- shared counters
struct InsertCounters {
  unsigned long long forward_accepted, forward_rejected, reverse_accepted, reverse_rejected;
  unsigned long long evictions_necessary, evictions_redundant, forced_links, n_requests;
};

// ------------------------------------------------------------- forward stage
// Warp per fresh node (slot start + i): union of in-bucket candidates (phys,
// f64) and search results (slot, f64) -> sort by (dist, slot) -> dedup ->
// nearest pre-batch -> greedy Eq.1/Eq.2 selection -> forward row + requests.
#ifndef GRAB_INSERT_MINB
#define GRAB_INSERT_MINB 6
#endif
// (128 threads, >= GRAB_INSERT_MINB blocks/SM: <= 80 registers for NC <= 2, so
// 24 warps per SM hide the row-load latency: forward 16.9 -> 14.6 ms at cfg2;
// wide rows keep their registers. k_rewire spills at 80-96 and stays at 128.)
template <int NC>
__global__ void __launch_bounds__(128, NC <= 2 ? GRAB_INSERT_MINB : 1) k_forward(uint64_t start, uint64_t b, const uint32_t* s2p, const Attr* attr, const int32_t* i2b,
                          const float* X, uint32_t dp, uint32_t* adj, uint32_t K, const uint32_t* loc_ids,
                          const double* loc_d, uint32_t KL, const int64_t* found_slots, const double* found_d,
                          const uint32_t* found_cnt, uint32_t KS, double alpha2, uint32_t P,
                          unsigned long long* req_key, double* req_d, uint32_t* nearest_pre, InsertCounters* cnt) {
  extern __shared__ __align__(16) uint8_t smem[];
  const uint32_t wib = threadIdx.x >> 5, lane = lane_id(), wpb = blockDim.x >> 5;
  const uint64_t i = blockIdx.x * (uint64_t)wpb + wib;
  if (i >= b) return;
  double* cd = (double*)smem + (uint64_t)wib * P;
  double* near = (double*)smem + (uint64_t)wpb * P + (uint64_t)wib * P;
  double* acc_d = (double*)smem + 2ull * wpb * P + (uint64_t)wib * K;                 // accepted dists (K)
  uint32_t* cs = (uint32_t*)((double*)smem + 2ull * wpb * P + (uint64_t)wpb * K) + (uint64_t)wib * P;  // slot
  uint32_t* acc_s = (uint32_t*)((double*)smem + 2ull * wpb * P + (uint64_t)wpb * K) + (uint64_t)wpb * P +
                    (uint64_t)wib * K;  // accepted slots (K)
  uint32_t* cph = (uint32_t*)((double*)smem + 2ull * wpb * P + (uint64_t)wpb * K) + (uint64_t)wpb * (P + K) +
                  (uint64_t)wib * P;  // phys of each candidate (P): row loads need no slot2phys gather
  uint16_t* alv = (uint16_t*)((uint32_t*)((double*)smem + 2ull * wpb * P + (uint64_t)wpb * K) +
                              (uint64_t)wpb * (2 * P + K)) + (uint64_t)wib * P;  // live tail indices (P)
  const uint64_t q = start + i;
  const uint32_t pq = s2p[q];
  // gather candidates
  uint32_t n = 0;
  for (uint32_t j = lane; j < P; j += 32) {
    cd[j] = __longlong_as_double(0x7FF0000000000000ll);
    cs[j] = kSentinel;
    cph[j] = 0;
  }
  __syncwarp();
  for (uint32_t j = lane; j < KL; j += 32) {
    uint32_t c = loc_ids[(uint64_t)pq * KL + j];
    if (c != kSentinel) {
      cd[j] = loc_d[(uint64_t)pq * KL + j];
      cs[j] = attr[c].slot;
      cph[j] = c;
    }
  }
  const uint32_t nf = found_cnt ? found_cnt[i] : 0;
  for (uint32_t j = lane; j < nf; j += 32) {
    cd[KL + j] = found_d[i * KS + j];
    const uint32_t sj = (uint32_t)found_slots[i * KS + j];
    cs[KL + j] = sj;
    cph[KL + j] = s2p[sj];
  }
  __syncwarp();
  // bitonic sort by (dist, slot)
  for (uint32_t k = 2; k <= P; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t t = lane; t < P; t += 32) {
        uint32_t l = t ^ j;
        if (l > t) {
          bool asc = (t & k) == 0;
          bool gt = key_less(cd[l], cs[l], cd[t], cs[t]);
          if (gt == asc) {
            double td = cd[t];
            cd[t] = cd[l];
            cd[l] = td;
            uint32_t ts = cs[t];
            cs[t] = cs[l];
            cs[l] = ts;
            ts = cph[t];
            cph[t] = cph[l];
            cph[l] = ts;
          }
        }
      }
      __syncwarp();
    }
  }
  // dedup (a slot found by both sources carries identical f64 distance bits):
  // flags from the unmodified array first, then an order-preserving compaction
  uint32_t keep_bits = 0;
  for (uint32_t c = 0; c * 32 < P; ++c) {
    uint32_t t = c * 32 + lane;
    if (cs[t] != kSentinel && (t == 0 || cs[t] != cs[t - 1])) keep_bits |= 1u << c;
  }
  __syncwarp();
  for (uint32_t c = 0; c * 32 < P; ++c) {
    uint32_t t = c * 32 + lane;
    bool keep = (keep_bits >> c) & 1u;
    uint32_t m = __ballot_sync(0xFFFFFFFFu, keep);
    double dv = cd[t];
    uint32_t sv = cs[t], pv = cph[t];
    __syncwarp();
    if (keep) {
      uint32_t pos = n + __popc(m & ((1u << lane) - 1));
      cd[pos] = dv;
      cs[pos] = sv;
      cph[pos] = pv;
    }
    n += __popc(m);
    __syncwarp();
  }
  if (n == 0) {
    if (lane == 0) nearest_pre[i] = kSentinel;
    return;
  }
  // nearest pre-batch node (updater.py:225-228)
  uint32_t npre = kSentinel;
  for (uint32_t t0 = 0; t0 < n && npre == kSentinel; t0 += 32) {
    uint32_t t = t0 + lane;
    uint32_t m = __ballot_sync(0xFFFFFFFFu, t < n && cs[t] < start);
    if (m) npre = cs[t0 + __ffs(m) - 1];
  }
  if (lane == 0) nearest_pre[i] = npre;
  // greedy selection (select_neighbors)
  for (uint32_t t = lane; t < n; t += 32) near[t] = __longlong_as_double(0x7FF0000000000000ll);
  __syncwarp();
  uint32_t nacc = 0;
  for (uint32_t t = 0; t < n && nacc < K; ++t) {
    const uint32_t s = cs[t];
    if (s == (uint32_t)q) continue;
    const double d = cd[t];
    const double de = s >= start ? alpha2 * d : d;
    if (!(de < near[t])) continue;
    if (lane == 0) {
      acc_s[nacc] = s;
      acc_d[nacc] = d;
    }
    ++nacc;
    // nearest_kept[j] = min(nearest_kept[j], dist(s, cand j)) for the undecided
    // tail. Only LIVE tail candidates are measured: j with de_j >= nearest_kept[j]
    // is already rejected whatever happens later (nearest_kept only decreases),
    // and self is never accepted, so skipping them changes no decision.
    RowRegs<NC> r;
    load_row<NC>(r, X, dp, cph[t]);
    uint32_t na = 0;
    for (uint32_t j0 = t + 1; j0 < n; j0 += 32) {
      const uint32_t j = j0 + lane;
      bool live = false;
      if (j < n) {
        const uint32_t sj = cs[j];
        const double dj = cd[j];
        const double dej = sj >= start ? alpha2 * dj : dj;
        live = sj != (uint32_t)q && dej < near[j];
      }
      const uint32_t m = __ballot_sync(0xFFFFFFFFu, live);
      if (live) alv[na + __popc(m & ((1u << lane) - 1))] = (uint16_t)j;
      na += __popc(m);
    }
    __syncwarp();
    {
      // near[j] only ever meets de_j (live iff de_j < near[j]), so what a
      // measurement must decide is dist(s, j) <= de_j. G rows per round are
      // screened in f32 (half the FP64 work); a row whose screen value is
      // within the error bound of de_j is re-measured exactly (row_dist: the
      // f64 tree) -- the decisions, and so the rows, are the f64 ones.
      constexpr int G = Batch<NC>::G, SH = Batch<NC>::SH;
      const double rel = screen_rel(dp);
      for (uint32_t a0 = 0; a0 < na; a0 += G) {
        uint32_t p[G];
        bool ok[G];
#pragma unroll
        for (int g = 0; g < G; ++g) {
          ok[g] = a0 + g < na;
          p[g] = ok[g] ? cph[alv[a0 + g]] : 0u;
        }
        const float fsum = dist_batch_f32<NC>(r, X, dp, p, ok);
        const uint32_t a = a0 + (lane >> SH);
        bool unsure = false;
        if ((lane & ((1u << SH) - 1)) == 0 && a < na) {
          const uint32_t j = alv[a];
          const double dj = cd[j];
          const double dej = cs[j] >= start ? alpha2 * dj : dj;
          const double f = (double)fsum, m = rel * fmax(f, dej);
          if (f < dej - m)
            near[j] = 0.0;  // dist <= de_j: j is rejected
          else if (!(f > dej + m))
            unsure = true;  // (else dist > de_j: no decision changes)
        }
        uint32_t um = __ballot_sync(0xFFFFFFFFu, unsure);
        while (um) {  // exact re-measure of the close calls, one row at a time
          const uint32_t src = __ffs(um) - 1;
          um &= um - 1;
          const uint32_t j = alv[a0 + (src >> SH)];
          const double d = row_dist<NC>(r, X, dp, cph[j]);
          if (lane == 0 && d < near[j]) near[j] = d;
        }
      }
    }
    __syncwarp();
  }
  __syncwarp();
  if (lane == 0) {
    atomicAdd(&cnt->forward_accepted, (unsigned long long)nacc);
    atomicAdd(&cnt->forward_rejected, (unsigned long long)(n - nacc));
  }
  // forward row: intra-bucket accepts first, then cross (updater.py:236-240)
  const int32_t bq = i2b[q];
  uint32_t* row = adj + (uint64_t)pq * K;
  if (lane == 0) {
    uint32_t col = 0;
    for (int pass = 0; pass < 2; ++pass)
      for (uint32_t j = 0; j < nacc; ++j) {
        uint32_t s = acc_s[j];
        bool intra = i2b[s] == bq;
        if ((pass == 0) == intra) {
          row[col] = s2p[s];  // (acc_s holds slots; one gather per accepted edge)
          // reverse request (v, q, d_vq) with the candidate distance
          req_key[i * K + col] = ((unsigned long long)s << 32) | (unsigned long long)q;
          req_d[i * K + col] = acc_d[j];
          ++col;
        }
      }
  }
}

// ------------------------------------------------------------- reverse stage
__global__ void k_req_heads(const unsigned long long* keys, uint64_t n, uint8_t* head) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  head[i] = (i == 0 || (keys[i] >> 32) != (keys[i - 1] >> 32)) ? 1 : 0;
}

// Sorted keys with an all-ones padding suffix: *nvalid = length of the valid
// prefix (the one index whose successor is padding), and head[i] = 1 where a
// run of equal high 32 bits starts inside that prefix (0 elsewhere).
__global__ void k_valid_heads(const unsigned long long* keys, uint64_t n, uint8_t* head, uint32_t* nvalid) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const bool v = keys[i] != ~0ull;
  if (v && (i + 1 == n || keys[i + 1] == ~0ull)) *nvalid = (uint32_t)(i + 1);
  if (i == 0 && !v) *nvalid = 0;
  head[i] = v && (i == 0 || (keys[i] >> 32) != (keys[i - 1] >> 32)) ? 1 : 0;
}

struct IsZero {
  const uint32_t* c;
  __host__ __device__ bool operator()(uint32_t i) const { return c[i] == 0; }
};
struct IsSet {
  const uint8_t* f;
  __host__ __device__ bool operator()(uint32_t i) const { return f[i] != 0; }
};

// Distances from the row in `r` to row entries j0 .. j0+G-1 of a lane-distributed
// row (entry j held by lane j % 32 in e[j / 32]), G = Batch<NC>::G rows in
// flight; entry j0 + g's distance is returned on lanes g << SH .. (g+1) << SH - 1
// (SENTINEL / j >= K: +inf). Bit-identical to row_dist (reduce_scatter pairs
// like warp_sum).
template <int NC>
__device__ __forceinline__ double dist_entries(const RowRegs<NC>& r, const float* X, uint32_t dp,
                                               const uint32_t (&e)[2], uint32_t j0, uint32_t K) {
  constexpr int G = Batch<NC>::G;
  const uint32_t lane = lane_id();
  uint32_t p[G];
  bool ok[G];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const uint32_t j = j0 + g;
    p[g] = __shfl_sync(0xFFFFFFFFu, (j & 32) ? e[1] : e[0], j & 31);
    ok[g] = j < K && p[g] != kSentinel;
  }
  const double sum = dist_batch<NC>(r, X, dp, p, ok);
  bool okl = false;
#pragma unroll
  for (int g = 0; g < G; ++g) okl = (lane >> Batch<NC>::SH) == (uint32_t)g ? ok[g] : okl;
  return okl ? sum : __longlong_as_double(0x7FF0000000000000ll);
}

// try_rewire for every request of one target v, in q order (updater.py:87-123).
// The row, and the distances from v to its eviction region, live in registers
// (entry j on lane j % 32, e[j / 32]; K <= 64): a request reads no row memory,
// the diversity test measures q against all K neighbours 8 rows per round
// (stopping at the first failing round), and an accepted q's distance to v is
// the request's own d_vq (the same f64 bits a recomputation gives).
template <int NC>
__global__ void k_rewire(const unsigned long long* keys, const double* dvq, uint64_t nreq, const uint32_t* heads,
                         uint32_t nheads, const uint32_t* s2p, const Attr* attr, const float* X, uint32_t dp,
                         uint32_t* adj, uint32_t K, uint32_t k_local, double alpha2, uint8_t* rewired_slot,
                         InsertCounters* cnt) {
  const uint32_t wib = threadIdx.x >> 5, lane = lane_id(), wpb = blockDim.x >> 5;
  const uint64_t h = blockIdx.x * (uint64_t)wpb + wib;
  if (h >= nheads) return;
  const uint64_t b0 = heads[h], b1 = h + 1 < nheads ? heads[h + 1] : nreq;
  const uint32_t v = (uint32_t)(keys[b0] >> 32);
  const uint32_t pv = s2p[v];
  uint32_t* row = adj + (uint64_t)pv * K;
  unsigned long long acc = 0, rej = 0, ev_nec = 0, ev_red = 0;
  const double kNegInf = -__longlong_as_double(0x7FF0000000000000ll);
  const uint32_t r0 = K > k_local ? k_local : 0;
  uint32_t e[2];
  double dv[2] = {kNegInf, kNegInf};  // distance to v, region entries only
  bool have_dv = false;                // computed lazily at the first eviction
#pragma unroll
  for (int u = 0; u < 2; ++u) e[u] = lane + 32 * u < K ? row[lane + 32 * u] : 0u;
  for (uint64_t r = b0; r < b1; ++r) {
    const uint32_t q = (uint32_t)keys[r];
    const uint32_t pq = s2p[q];
    const bool in0 = lane < K, in1 = lane + 32 < K;
    if (__any_sync(0xFFFFFFFFu, (in0 && e[0] == pq) || (in1 && e[1] == pq))) {  // duplicate
      ++rej;
      continue;
    }
    const uint32_t f0 = __ballot_sync(0xFFFFFFFFu, in0 && e[0] == kSentinel);
    const uint32_t f1 = __ballot_sync(0xFFFFFFFFu, in1 && e[1] == kSentinel);
    int32_t pos = -1;
    if (f0 | f1) {
      pos = f0 ? __ffs(f0) - 1 : 32 + __ffs(f1) - 1;
    } else {
      // Eq.1/Eq.2 diversity test against every current neighbour
      const double deff = alpha2 * dvq[r];
      RowRegs<NC> rq;
      load_row<NC>(rq, X, dp, pq);
      bool ok = true;
      constexpr int G = Batch<NC>::G, SH = Batch<NC>::SH;
      const double rel = screen_rel(dp);
      // reject iff some neighbour n has dist(q, n) <= deff: screened in f32,
      // rows within the error bound of deff re-measured exactly (f64 tree)
      for (uint32_t j0 = 0; j0 < K && ok; j0 += G) {
        uint32_t p[G];
        bool okg[G];
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const uint32_t j = j0 + g;
          p[g] = __shfl_sync(0xFFFFFFFFu, (j & 32) ? e[1] : e[0], j & 31);
          okg[g] = j < K && p[g] != kSentinel;
        }
        const float f = dist_batch_f32<NC>(rq, X, dp, p, okg);
        bool okl = false;
        uint32_t pl = 0;
#pragma unroll
        for (int g = 0; g < G; ++g) {
          okl = (lane >> SH) == (uint32_t)g ? okg[g] : okl;
          pl = (lane >> SH) == (uint32_t)g ? p[g] : pl;
        }
        bool fail = false, unsure = false;
        if ((lane & ((1u << SH) - 1)) == 0 && okl) {
          const double fd = (double)f, m = rel * fmax(fd, deff);
          if (fd < deff - m)
            fail = true;
          else if (!(fd > deff + m))
            unsure = true;
        }
        if (__any_sync(0xFFFFFFFFu, fail)) {
          ok = false;
          break;
        }
        uint32_t um = __ballot_sync(0xFFFFFFFFu, unsure);
        while (um && ok) {
          const uint32_t src = __ffs(um) - 1;
          um &= um - 1;
          const double d = row_dist<NC>(rq, X, dp, __shfl_sync(0xFFFFFFFFu, pl, src));
          ok = deff < d;
        }
      }
      if (!ok) {
        ++rej;
        continue;
      }
      if (!have_dv) {
        have_dv = true;
        RowRegs<NC> rv;  // v's row is needed only here (q's diversity test is done)
        load_row<NC>(rv, X, dp, pv);
        for (uint32_t j0 = r0; j0 < K; j0 += G) {
          const double dj = dist_entries<NC>(rv, X, dp, e, j0, K);
#pragma unroll
          for (int g = 0; g < G; ++g) {
            const double dg = __shfl_sync(0xFFFFFFFFu, dj, g << SH);
            const uint32_t j = j0 + g;
            if (j < K && lane == (j & 31)) {
              if (j & 32)
                dv[1] = dg;
              else
                dv[0] = dg;
            }
          }
        }
      }
      // farthest neighbour of v in the region, first index on ties
      double bd = kNegInf;
      int32_t bp = 0x7FFFFFFF;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const uint32_t j = lane + 32 * u;
        if (j >= r0 && j < K && (dv[u] > bd || (dv[u] == bd && (int32_t)j < bp))) {
          bd = dv[u];
          bp = (int32_t)j;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double od = __shfl_xor_sync(0xFFFFFFFFu, bd, o);
        const int32_t op = __shfl_xor_sync(0xFFFFFFFFu, bp, o);
        if (od > bd || (od == bd && op < bp)) {
          bd = od;
          bp = op;
        }
      }
      pos = bp;
      if ((uint32_t)pos >= k_local)
        ++ev_red;
      else
        ++ev_nec;
    }
    if (lane == (uint32_t)(pos & 31)) {
      if (pos & 32) {
        e[1] = pq;
        dv[1] = dvq[r];
      } else {
        e[0] = pq;
        dv[0] = dvq[r];
      }
    }
    if (lane == 0) row[pos] = pq;
    __syncwarp();
    ++acc;
  }
  if (lane == 0) {
    atomicAdd(&cnt->reverse_accepted, acc);
    atomicAdd(&cnt->reverse_rejected, rej);
    atomicAdd(&cnt->evictions_necessary, ev_nec);
    atomicAdd(&cnt->evictions_redundant, ev_red);
    if (acc) rewired_slot[v] = 1;
  }
}

// ------------------------------------------------------------- heal stage
__global__ void k_prefix_indeg(const uint32_t* adj, const uint32_t* s2p, const Attr* attr, uint64_t prefix,
                               uint32_t K, uint64_t start, uint64_t end, uint32_t* counts) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= prefix * K) return;
  uint32_t v = adj[(uint64_t)s2p[i / K] * K + i % K];
  if (v == kSentinel) return;
  uint32_t s = attr[v].slot;
  if (s >= start && s < end) atomicAdd(counts + (s - start), 1u);
}

// _heal_unreachable decisions: the target row v of a missing newcomer q depends
// only on q's own (fresh, unchanging) row and nearest_pre, so all choices are
// made in parallel; rows v are then patched serially per v, in q order.
template <int NC>
__global__ void k_heal_choose(const uint32_t* missing, uint32_t nmiss, uint64_t start, const uint32_t* s2p,
                              const Attr* attr, const float* X, uint32_t dp, const uint32_t* adj, uint32_t K,
                              const uint32_t* nearest_pre, unsigned long long* keys) {
  const uint32_t wib = threadIdx.x >> 5, wpb = blockDim.x >> 5;
  const uint64_t t = blockIdx.x * (uint64_t)wpb + wib;
  if (t >= nmiss) return;
  const uint64_t q = start + missing[t];
  const uint32_t pq = s2p[q];
  const uint32_t* rq = adj + (uint64_t)pq * K;
  RowRegs<NC> qr;
  load_row<NC>(qr, X, dp, pq);
  double bd = __longlong_as_double(0x7FF0000000000000ll);
  uint32_t v = kSentinel;
  for (uint32_t j = 0; j < K; ++j) {
    const uint32_t e = rq[j];
    if (e == kSentinel) continue;
    const uint32_t s = attr[e].slot;
    if (s >= start) continue;
    const double d = row_dist<NC>(qr, X, dp, e);
    if (key_less(d, s, bd, v)) {
      bd = d;
      v = s;
    }
  }
  if (v == kSentinel) v = nearest_pre[missing[t]];
  if (lane_id() == 0) keys[t] = v == kSentinel ? ~0ull : (((unsigned long long)v << 32) | (unsigned long long)q);
}

// Forced links into one target row v, requests in q order (updater.py:301-321).
// The row's entries, their f64 distances to v and their "stale" flag (slot
// outside the batch) are cached per lane (entries j = lane, lane + 32; K <= 64)
// once, so a request costs one distance (the new entry's) instead of
// re-measuring the whole eviction region; eviction = first argmax of the
// cached distance over [K_local, K), stale entries preferred.
template <int NC>
__global__ void k_heal_apply(const unsigned long long* keys, uint64_t nreq, const uint32_t* heads, uint32_t nheads,
                             uint64_t start, uint64_t end, const uint32_t* s2p, const Attr* attr, const float* X,
                             uint32_t dp, uint32_t* adj, uint32_t K, uint32_t k_local, uint8_t* rewired_slot,
                             InsertCounters* cnt) {
  const uint32_t wib = threadIdx.x >> 5, lane = lane_id(), wpb = blockDim.x >> 5;
  const uint64_t h = blockIdx.x * (uint64_t)wpb + wib;
  if (h >= nheads) return;
  const uint64_t b0 = heads[h], b1 = h + 1 < nheads ? heads[h + 1] : nreq;
  const uint32_t v = (uint32_t)(keys[b0] >> 32);
  const uint32_t pv = s2p[v];
  uint32_t* row = adj + (uint64_t)pv * K;
  RowRegs<NC> vr;
  load_row<NC>(vr, X, dp, pv);
  const double kNegInf = -__longlong_as_double(0x7FF0000000000000ll);
  uint32_t e[2];
  double d[2];
  bool st[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const uint32_t j = lane + 32 * u;
    e[u] = j < K ? row[j] : kSentinel;
    st[u] = false;
    if (e[u] != kSentinel) {
      const uint32_t s = attr[e[u]].slot;
      st[u] = s < start || s >= end;
    }
  }
  const uint32_t r0 = K > k_local ? k_local : 0;
  // distances of the current eviction-region entries [r0, K): G rows in flight
  // per round (same reduction tree as row_dist); empty entries keep -inf
  d[0] = d[1] = kNegInf;
  constexpr int G = Batch<NC>::G, SH = Batch<NC>::SH;
  for (uint32_t j0 = r0; j0 < K; j0 += G) {
    const double sum = dist_entries<NC>(vr, X, dp, e, j0, K);
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const double dg = __shfl_sync(0xFFFFFFFFu, sum, g << SH);
      const uint32_t j = j0 + g;
      const uint32_t eo = __shfl_sync(0xFFFFFFFFu, (j & 32) ? e[1] : e[0], j & 31);
      if (j < K && eo != kSentinel && lane == (j & 31)) {
        if (j & 32)
          d[1] = dg;
        else
          d[0] = dg;
      }
    }
  }
  unsigned long long forced = 0, evict = 0;
  for (uint64_t r = b0; r < b1; ++r) {
    const uint32_t pq = s2p[(uint32_t)keys[r]];
    const uint32_t f0 = __ballot_sync(0xFFFFFFFFu, e[0] == kSentinel && lane < K);
    const uint32_t f1 = __ballot_sync(0xFFFFFFFFu, e[1] == kSentinel && lane + 32 < K);
    int32_t pos;
    if (f0 | f1) {
      pos = f0 ? __ffs(f0) - 1 : 32 + __ffs(f1) - 1;
    } else {
      // first argmax over the region, stale entries first
      int32_t best_pos = -1;
      double best_d = kNegInf;
      for (int pass = 0; pass < 2 && best_pos < 0; ++pass) {
        double bd = kNegInf;
        int32_t bp = 0x7FFFFFFF;
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const uint32_t j = lane + 32 * u;
          const bool in = j >= r0 && j < K && (pass == 1 || st[u]);
          if (in && (d[u] > bd || (d[u] == bd && (int32_t)j < bp))) {
            bd = d[u];
            bp = (int32_t)j;
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double od = __shfl_xor_sync(0xFFFFFFFFu, bd, o);
          const int32_t op = __shfl_xor_sync(0xFFFFFFFFu, bp, o);
          if (od > bd || (od == bd && op < bp)) {
            bd = od;
            bp = op;
          }
        }
        if (bp != 0x7FFFFFFF) {
          best_pos = bp;
          best_d = bd;
        }
      }
      (void)best_d;
      pos = best_pos;
      ++evict;
    }
    const double dq = row_dist<NC>(vr, X, dp, pq);
    if (lane == (uint32_t)(pos & 31)) {
      const int u = pos >> 5;
      if (u == 0) {
        e[0] = pq;
        d[0] = dq;
        st[0] = false;
      } else {
        e[1] = pq;
        d[1] = dq;
        st[1] = false;
      }
    }
    if (lane == 0) row[pos] = pq;
    __syncwarp();
    ++forced;
  }
  if (lane == 0) {
    atomicAdd(&cnt->forced_links, forced);
    atomicAdd(&cnt->evictions_redundant, evict);
    rewired_slot[v] = 1;
  }
}

// Sorted u64 keys (valid prefix, ~0 padding) -> number of valid keys and the
// start index of every run with equal high 32 bits (one host round trip).
static uint64_t segment_heads(Pool& pool, const unsigned long long* keys, uint64_t n, uint32_t** heads_out,
                              uint32_t* nheads_out, cudaStream_t st) {
  *nheads_out = 0;
  if (!n) return 0;
  uint8_t* head = pool.alloc<uint8_t>(n);
  uint32_t* cnts = pool.alloc<uint32_t>(2);  // {nvalid, nheads}
  k_valid_heads<<<(unsigned)div_up(n, 256), 256, 0, st>>>(keys, n, head, cnts);
  GRAB_CHECK_LAUNCH();
  uint32_t* heads = pool.alloc<uint32_t>(n);
  cub::CountingInputIterator<uint32_t> idx(0);
  size_t tmp = 0;
  cub::DeviceSelect::Flagged(nullptr, tmp, idx, head, heads, cnts + 1, (int)n, st);
  void* t = pool.alloc<uint8_t>(tmp);
  GRAB_CUDA(cub::DeviceSelect::Flagged(t, tmp, idx, head, heads, cnts + 1, (int)n, st));
  uint32_t hc[2];
  GRAB_CUDA(cudaMemcpyAsync(hc, cnts, 8, cudaMemcpyDeviceToHost, st));
  GRAB_CUDA(cudaStreamSynchronize(st));
  *heads_out = heads;
  *nheads_out = hc[1];
  return hc[0];
}

static unsigned long long* sort_keys(Pool& pool, unsigned long long* keys, uint64_t n, cudaStream_t st) {
  unsigned long long* out = pool.alloc<unsigned long long>(n);
  size_t tmp = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, tmp, keys, out, (int)n, 0, 64, st);
  void* t = pool.alloc<uint8_t>(tmp);
  GRAB_CUDA(cub::DeviceRadixSort::SortKeys(t, tmp, keys, out, (int)n, 0, 64, st));
  return out;
}

// ------------------------------------------------------------- driver
template <class F>
static void by_nc(uint32_t dp, F&& f) {
  uint32_t nc = (uint32_t)div_up(dp, 128);
  if (nc <= 1)
    f(std::integral_constant<int, 1>{});
  else if (nc <= 2)
    f(std::integral_constant<int, 2>{});
  else if (nc <= 4)
    f(std::integral_constant<int, 4>{});
  else if (nc <= 8)
    f(std::integral_constant<int, 8>{});
  else if (nc <= 16)
    f(std::integral_constant<int, 16>{});
  else
    throw Error(GRAB_ERR_VALUE, "dimension > 2048 not supported");
}

__global__ void k_fresh_phys(const uint32_t* s2p, uint64_t start, uint64_t b, uint32_t* out) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i < b) out[i] = s2p[start + i];
}

// append_batch (layout.py:181-223) alone: rows, scalars, ids and bucket maps at
// the tail (zero-shift slab placement), adjacency left SENTINEL; [start, end).
void append_batch_device(DevIndex& ix, const float* vectors, const float* scalars, const int64_t* ids, uint64_t b,
                         uint32_t mem, uint64_t* start_out, uint64_t* end_out) {
  cudaStream_t st = ix.stream;
  const uint64_t n0 = ix.count;
  if (start_out) *start_out = n0;
  if (end_out) *end_out = n0;
  if (b == 0) return;
  if (!ix.built) throw Error(GRAB_ERR_STATE, "index has no bucket metadata (build it first)");
  if (n0 + b > ix.n_cap)
    throw Error(GRAB_ERR_CAPACITY, "capacity exhausted: " + std::to_string(n0) + " claimed + " + std::to_string(b) +
                                       " requested > " + std::to_string(ix.n_cap));
  Pool pool(st);
  const float* Vd = vectors;
  const float* Sd = scalars;
  if (mem == GRAB_MEM_HOST) {
    for (uint64_t i = 0; i < b; ++i)
      if (!std::isfinite(scalars[i])) throw Error(GRAB_ERR_VALUE, "scalars must be finite");
    float* v = pool.alloc<float>(b * ix.dim);
    float* sc = pool.alloc<float>(b);
    GRAB_CUDA(cudaMemcpyAsync(v, vectors, b * ix.dim * 4, cudaMemcpyHostToDevice, st));
    GRAB_CUDA(cudaMemcpyAsync(sc, scalars, b * 4, cudaMemcpyHostToDevice, st));
    Vd = v;
    Sd = sc;
  }
  launch_bucket_ids(ix, Sd, b, ix.i2b + n0, st);
  layout_append(ix, Vd, Sd, n0, b);
  for (uint64_t i = 0; i < b; ++i) ix.ids[n0 + i] = ids ? ids[i] : (int64_t)(n0 + i);
  GRAB_CUDA(cudaStreamSynchronize(st));
  if (end_out) *end_out = n0 + b;
}

void insert_batch_device(DevIndex& ix, const float* vectors, const float* scalars, const int64_t* ids, uint64_t b,
                         uint32_t search_itopk, uint32_t mem, grab_insert_report* rep) {
  const double t_begin = now_s();
  cudaStream_t st = ix.stream;
  grab_insert_report R{};
  R.batch_size = b;
  ix.last_rewired.clear();
  Pool pool(st);
  // stage rows on the device
  const float* Vd = vectors;
  const float* Sd = scalars;
  if (b && mem == GRAB_MEM_HOST) {
    for (uint64_t i = 0; i < b; ++i)
      if (!std::isfinite(scalars[i])) throw Error(GRAB_ERR_VALUE, "scalars must be finite");
    float* v = pool.alloc<float>(b * ix.dim);
    float* s = pool.alloc<float>(b);
    GRAB_CUDA(cudaMemcpyAsync(v, vectors, b * ix.dim * 4, cudaMemcpyHostToDevice, st));
    GRAB_CUDA(cudaMemcpyAsync(s, scalars, b * 4, cudaMemcpyHostToDevice, st));
    Vd = v;
    Sd = s;
  }
  // empty index: bulk-build the first bucket_capacity rows (updater.py:175-189)
  if (ix.count == 0) {
    if (b == 0) {
      if (rep) *rep = R;
      return;
    }
    uint64_t head = std::min<uint64_t>(b, ix.params.bucket_capacity);
    // the reference bulk-builds through build_index, which ignores ids: the head
    // keeps ids = arange(head) (build_index_device sets them); only ids[head:]
    // reach the appended tail (updater.py:175-189)
    build_index_device(ix, Vd, Sd, head, GRAB_STRATEGY_QUANTILE, ix.params.k_max, 3, GRAB_MEM_DEVICE, nullptr);
    R.bulk_built = head;
    if (head == b) {
      R.wall_time_s = now_s() - t_begin;
      if (rep) *rep = R;
      return;
    }
    Vd += head * ix.dim;
    Sd += head;
    if (ids) ids += head;
    b -= head;
  }
  if (b == 0) {
    R.wall_time_s = now_s() - t_begin;
    if (rep) *rep = R;
    return;
  }
  if (!ix.built) throw Error(GRAB_ERR_STATE, "index has no bucket metadata");
  const uint64_t n0 = ix.count;
  if (n0 + b > ix.n_cap)
    throw Error(GRAB_ERR_CAPACITY, "capacity exhausted: " + std::to_string(n0) + " claimed + " + std::to_string(b) +
                                       " requested > " + std::to_string(ix.n_cap));
  const uint64_t start = n0, end = n0 + b;
  const uint32_t K = ix.params.k_max;
  double tp = now_s();
  auto mark = [&](int ph) {
    GRAB_CUDA(cudaStreamSynchronize(st));
    double t = now_s();
    R.phase_seconds[ph] += t - tp;
    tp = t;
  };
  // ---- append (bucket ids, zero-shift placement)
  launch_bucket_ids(ix, Sd, b, ix.i2b + start, st);
  std::vector<uint32_t> old_count = ix.h_bcount;
  layout_append(ix, Vd, Sd, start, b);
  for (uint64_t i = 0; i < b; ++i) ix.ids[start + i] = ids ? ids[i] : (int64_t)(start + i);

  mark(0);
  // ---- in-bucket candidates: causal kNN over each touched slab (run beside the
  // candidate search on a second stream it gains nothing: the search grid holds
  // every SM and the screen needs a whole SM's shared memory; measured)
  const uint32_t KL = 2 * K;
  uint32_t* loc_ids = pool.alloc<uint32_t>(ix.phys_cap * (uint64_t)KL);
  double* loc_d = pool.alloc<double>(ix.phys_cap * (uint64_t)KL);
  GRAB_CUDA(cudaMemsetAsync(loc_ids, 0xFF, ix.phys_cap * (uint64_t)KL * 4, st));
  {
    float* norms = pool.alloc<float>(ix.phys_cap);
    row_norms(ix, norms, st);
    std::vector<KnnJob> jobs;
    for (uint32_t k = 0; k < ix.m; ++k) {
      uint32_t s0 = ix.h_bstart[k], c_old = old_count[k], c_new = ix.h_bcount[k];
      for (uint32_t r = c_old; r < c_new; r += kKnnBM)
        jobs.push_back({s0 + r, std::min<uint32_t>(kKnnBM, c_new - r), s0, s0 + c_new});
    }
    knn_device(ix, norms, jobs, KL, /*tb_slot=*/false, loc_ids, loc_d, st, /*causal=*/true);
  }
  mark(1);
  // ---- full-range graph search over the pre-batch prefix
  const uint32_t KS = search_itopk;
  int64_t* found_slots = nullptr;
  double* found_d = nullptr;
  uint32_t* found_cnt = nullptr;
  uint32_t* fresh_phys = pool.alloc<uint32_t>(b);
  k_fresh_phys<<<(unsigned)div_up(b, 256), 256, 0, st>>>(ix.slot2phys, start, b, fresh_phys);
  GRAB_CHECK_LAUNCH();
  if (n0 > 0) {
    found_slots = pool.alloc<int64_t>(b * KS);
    found_d = pool.alloc<double>(b * KS);
    found_cnt = pool.alloc<uint32_t>(b);
    double* lo = pool.alloc<double>(1);
    double* hi = pool.alloc<double>(1);
    const double inf = INFINITY, ninf = -INFINITY;
    GRAB_CUDA(cudaMemcpyAsync(lo, &ninf, 8, cudaMemcpyHostToDevice, st));
    GRAB_CUDA(cudaMemcpyAsync(hi, &inf, 8, cudaMemcpyHostToDevice, st));
    SearchArgs a{};
    a.X = ix.X;
    a.attr = ix.attr;
    a.adj = ix.adj;
    a.dp = ix.dp;
    a.k_max = K;
    a.bound = ix.bound;
    a.m = ix.m;
    a.bstart = ix.bstart;
    a.bcount = ix.bcount;
    a.bcum = ix.bcum;
    a.n_live = n0;
    a.Q = nullptr;
    a.qphys = fresh_phys;
    a.lower = lo;
    a.upper = hi;
    a.range_stride = 0;
    a.seeds = nullptr;
    a.seed_base = ix.params.rng_seed;
    a.ordinal0 = start;
    a.k = KS;
    a.itopk = KS;
    a.width = 4;
    a.max_iter = 50;
    a.want = std::min<uint32_t>(KS, 32);
    a.nwork = (uint32_t)b;
    a.out_slots = found_slots;
    a.out_dists = found_d;
    a.out_counts = found_cnt;
    a.out_stats = nullptr;
    ix.adj_version++;  // append / relayout changed rows since the last search
    run_search(ix, a, st);
  }
  mark(2);
  // ---- forward selection
  const double alpha2 = ix.params.alpha * ix.params.alpha;
  InsertCounters* cnt = pool.alloc<InsertCounters>(1);
  GRAB_CUDA(cudaMemsetAsync(cnt, 0, sizeof(InsertCounters), st));
  unsigned long long* req_key = pool.alloc<unsigned long long>(b * K);
  double* req_d = pool.alloc<double>(b * K);
  GRAB_CUDA(cudaMemsetAsync(req_key, 0xFF, b * K * 8, st));
  uint32_t* nearest_pre = pool.alloc<uint32_t>(b);
  uint32_t P = 32;
  while (P < KL + (n0 > 0 ? KS : 0)) P <<= 1;
  {
    const uint32_t wpb = 4;
    size_t smem = (size_t)wpb * (P * (8 + 8 + 4 + 4 + 2) + K * (8 + 4));
    by_nc(ix.dp, [&](auto ncv) {
      constexpr int NC = decltype(ncv)::value;
      auto kern = k_forward<NC>;
      GRAB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      kern<<<(unsigned)div_up(b, wpb), 32 * wpb, smem, st>>>(start, b, ix.slot2phys, ix.attr, ix.i2b, ix.X, ix.dp,
                                                             ix.adj, K, loc_ids, loc_d, KL, found_slots, found_d,
                                                             found_cnt, KS, alpha2, P, req_key, req_d, nearest_pre,
                                                             cnt);
      GRAB_CHECK_LAUNCH();
    });
  }
  mark(3);
  // ---- reverse rewiring: sort requests by (v, q)
  uint8_t* rewired = pool.alloc<uint8_t>(ix.n_cap);
  GRAB_CUDA(cudaMemsetAsync(rewired, 0, ix.n_cap, st));
  {
    const uint64_t nr_all = b * K;
    unsigned long long* k2 = pool.alloc<unsigned long long>(nr_all);
    double* d2 = pool.alloc<double>(nr_all);
    size_t tmp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp, req_key, k2, req_d, d2, (int)nr_all, 0, 64, st);
    void* t = pool.alloc<uint8_t>(tmp);
    GRAB_CUDA(cub::DeviceRadixSort::SortPairs(t, tmp, req_key, k2, req_d, d2, (int)nr_all, 0, 64, st));
    // valid requests are the prefix (unused entries are all-ones keys): its length
    // and the per-target run heads in one pass, one host round trip for both counts
    uint32_t* heads = nullptr;
    uint32_t nheads = 0;
    const uint64_t nreq = segment_heads(pool, k2, nr_all, &heads, &nheads, st);
    if (nreq) {
      const uint32_t wpb = 4;
      by_nc(ix.dp, [&](auto ncv) {
        constexpr int NC = decltype(ncv)::value;
        k_rewire<NC><<<(unsigned)div_up(nheads, wpb), 32 * wpb, 0, st>>>(
            k2, d2, nreq, heads, nheads, ix.slot2phys, ix.attr, ix.X, ix.dp, ix.adj, K, ix.params.k_local, alpha2,
            rewired, cnt);
        GRAB_CHECK_LAUNCH();
      });
    }
  }
  mark(4);
  // ---- heal (n0 > 0)
  if (n0 > 0) {
    uint32_t* counts = pool.alloc<uint32_t>(b);
    uint32_t* miss = pool.alloc<uint32_t>(b);
    unsigned long long* hkeys = pool.alloc<unsigned long long>(b);
    uint32_t* nmiss_d = pool.alloc<uint32_t>(1);
    void* sel_tmp = nullptr;
    size_t sel_tmp_bytes = 0;
    for (int round = 0; round < 4; ++round) {
      GRAB_CUDA(cudaMemsetAsync(counts, 0, b * 4, st));
      k_prefix_indeg<<<(unsigned)div_up(start * K, 256), 256, 0, st>>>(ix.adj, ix.slot2phys, ix.attr, start, K, start,
                                                                       end, counts);
      GRAB_CHECK_LAUNCH();
      // newcomers without an in-edge from the prefix, compacted on the device
      {
        cub::CountingInputIterator<uint32_t> idx(0);
        size_t tmp = 0;
        cub::DeviceSelect::If(nullptr, tmp, idx, miss, nmiss_d, (int)b, IsZero{counts}, st);
        if (tmp > sel_tmp_bytes) {
          sel_tmp = pool.alloc<uint8_t>(tmp);
          sel_tmp_bytes = tmp;
        }
        GRAB_CUDA(cub::DeviceSelect::If(sel_tmp, tmp, idx, miss, nmiss_d, (int)b, IsZero{counts}, st));
      }
      uint32_t nm = 0;
      GRAB_CUDA(cudaMemcpyAsync(&nm, nmiss_d, 4, cudaMemcpyDeviceToHost, st));
      GRAB_CUDA(cudaStreamSynchronize(st));
      if (nm == 0) break;
      by_nc(ix.dp, [&](auto ncv) {
        constexpr int NC = decltype(ncv)::value;
        k_heal_choose<NC><<<(unsigned)div_up(nm, 4), 128, 0, st>>>(miss, nm, start, ix.slot2phys, ix.attr, ix.X,
                                                                    ix.dp, ix.adj, K, nearest_pre, hkeys);
        GRAB_CHECK_LAUNCH();
      });
      unsigned long long* sk = sort_keys(pool, hkeys, nm, st);
      uint32_t* heads = nullptr;
      uint32_t nheads = 0;
      const uint64_t nv = segment_heads(pool, sk, nm, &heads, &nheads, st);
      if (!nv) continue;
      by_nc(ix.dp, [&](auto ncv) {
        constexpr int NC = decltype(ncv)::value;
        k_heal_apply<NC><<<(unsigned)div_up(nheads, 4), 128, 0, st>>>(sk, nv, heads, nheads, start, end, ix.slot2phys,
                                                                      ix.attr, ix.X, ix.dp, ix.adj, K,
                                                                      ix.params.k_local, rewired, cnt);
        GRAB_CHECK_LAUNCH();
      });
    }
  }
  mark(5);
  InsertCounters hcnt;
  GRAB_CUDA(cudaMemcpyAsync(&hcnt, cnt, sizeof(hcnt), cudaMemcpyDeviceToHost, st));
  {  // rewired slots, ascending, compacted on the device
    uint32_t* rlist = pool.alloc<uint32_t>(end);
    uint32_t* nrw_d = pool.alloc<uint32_t>(1);
    cub::CountingInputIterator<uint32_t> idx(0);
    size_t tmp = 0;
    cub::DeviceSelect::If(nullptr, tmp, idx, rlist, nrw_d, (int)end, IsSet{rewired}, st);
    void* t = pool.alloc<uint8_t>(tmp);
    GRAB_CUDA(cub::DeviceSelect::If(t, tmp, idx, rlist, nrw_d, (int)end, IsSet{rewired}, st));
    uint32_t nrw = 0;
    GRAB_CUDA(cudaMemcpyAsync(&nrw, nrw_d, 4, cudaMemcpyDeviceToHost, st));
    GRAB_CUDA(cudaStreamSynchronize(st));
    ix.last_rewired.resize(nrw);
    if (nrw) GRAB_CUDA(cudaMemcpyAsync(ix.last_rewired.data(), rlist, (size_t)nrw * 4, cudaMemcpyDeviceToHost, st));
  }
  GRAB_CUDA(cudaStreamSynchronize(st));
  R.forward_accepted = hcnt.forward_accepted;
  R.forward_rejected = hcnt.forward_rejected;
  R.reverse_accepted = hcnt.reverse_accepted;
  R.reverse_rejected = hcnt.reverse_rejected;
  R.evictions_necessary = hcnt.evictions_necessary;
  R.evictions_redundant = hcnt.evictions_redundant;
  R.forced_links = hcnt.forced_links;
  R.n_rewired = ix.last_rewired.size();
  R.wall_time_s = now_s() - t_begin;
  if (rep) *rep = R;
}

// ------------------------------------------------------------- primitives
template <int NC>
__global__ void k_select_one(const float* X, uint32_t dp, int64_t target, const int64_t* cs, const double* cd,
                             const uint8_t* fresh, uint32_t n, uint32_t cap, double alpha2, double* near,
                             int64_t* out, uint32_t* nout) {
  const uint32_t lane = lane_id();
  for (uint32_t t = lane; t < n; t += 32) near[t] = __longlong_as_double(0x7FF0000000000000ll);
  __syncwarp();
  uint32_t nacc = 0;
  for (uint32_t t = 0; t < n && nacc < cap; ++t) {
    const int64_t s = cs[t];
    if (s == target) continue;
    bool dup = false;
    for (uint32_t j = 0; j < nacc; ++j) dup |= out[j] == s;
    if (dup) continue;
    const double de = fresh[t] ? alpha2 * cd[t] : cd[t];
    if (!(de < near[t])) continue;
    if (lane == 0) out[nacc] = s;
    ++nacc;
    RowRegs<NC> r;
    load_row<NC>(r, X, dp, (uint32_t)s);
    for (uint32_t j = 0; j < n; ++j) {
      double dj = row_dist<NC>(r, X, dp, (uint32_t)cs[j]);
      if (lane == 0 && dj < near[j]) near[j] = dj;
    }
    __syncwarp();
  }
  if (lane == 0) *nout = nacc;
}

template <int NC>
__global__ void k_rewire_one(const float* X, uint32_t dp, uint32_t* row, uint32_t K, uint32_t v, uint32_t q,
                             double dvq, double alpha2, uint32_t k_local, int32_t* res) {
  const uint32_t lane = lane_id();
  for (uint32_t j = 0; j < K; ++j)
    if (row[j] == q) {
      if (lane == 0) res[0] = 0, res[1] = -1;
      return;
    }
  for (uint32_t j = 0; j < K; ++j)
    if (row[j] == kSentinel) {
      if (lane == 0) row[j] = q, res[0] = 1, res[1] = -1;
      return;
    }
  RowRegs<NC> rq, rv;
  load_row<NC>(rq, X, dp, q);
  load_row<NC>(rv, X, dp, v);
  const double deff = alpha2 * dvq;
  for (uint32_t j = 0; j < K; ++j)
    if (!(deff < row_dist<NC>(rq, X, dp, row[j]))) {
      if (lane == 0) res[0] = 0, res[1] = -1;
      return;
    }
  const uint32_t r0 = K > k_local ? k_local : 0;
  double best = -1.0;
  int32_t pos = -1;
  for (uint32_t j = r0; j < K; ++j) {
    double d = row_dist<NC>(rv, X, dp, row[j]);
    if (d > best) best = d, pos = (int32_t)j;
  }
  if (lane == 0) row[pos] = q, res[0] = 1, res[1] = pos;
}

static float* upload_rows(const float* X, uint64_t n, uint32_t dim, uint32_t dp, cudaStream_t st) {
  float* d;
  GRAB_CUDA(cudaMallocAsync(&d, std::max<uint64_t>(n, 1) * dp * 4, st));
  GRAB_CUDA(cudaMemsetAsync(d, 0, n * dp * 4, st));
  GRAB_CUDA(cudaMemcpy2DAsync(d, dp * 4, X, dim * 4, dim * 4, n, cudaMemcpyHostToDevice, st));
  return d;
}

void select_neighbors_device(const float* X, uint64_t n_rows, uint32_t dim, int64_t target, const int64_t* cand_slots,
                             const double* cand_dists, const uint8_t* cand_fresh, uint32_t n_cand,
                             uint32_t row_capacity, double alpha, int64_t* out_accepted, uint32_t* n_accepted) {
  cudaStream_t st = 0;
  *n_accepted = 0;
  if (!n_cand) return;
  for (uint32_t i = 0; i < n_cand; ++i)
    if (cand_slots[i] < 0 || (uint64_t)cand_slots[i] >= n_rows) throw Error(GRAB_ERR_VALUE, "candidate slot out of range");
  const uint32_t dp = (dim + 3) / 4 * 4;
  float* dX = upload_rows(X, n_rows, dim, dp, st);
  Pool pool(st);
  int64_t* cs = pool.alloc<int64_t>(n_cand);
  double* cd = pool.alloc<double>(n_cand);
  uint8_t* fr = pool.alloc<uint8_t>(n_cand);
  double* near = pool.alloc<double>(n_cand);
  int64_t* out = pool.alloc<int64_t>(std::max<uint32_t>(row_capacity, 1));
  uint32_t* nout = pool.alloc<uint32_t>(1);
  GRAB_CUDA(cudaMemcpyAsync(cs, cand_slots, n_cand * 8, cudaMemcpyHostToDevice, st));
  GRAB_CUDA(cudaMemcpyAsync(cd, cand_dists, n_cand * 8, cudaMemcpyHostToDevice, st));
  GRAB_CUDA(cudaMemcpyAsync(fr, cand_fresh, n_cand, cudaMemcpyHostToDevice, st));
  by_nc(dp, [&](auto ncv) {
    constexpr int NC = decltype(ncv)::value;
    k_select_one<NC><<<1, 32, 0, st>>>(dX, dp, target, cs, cd, fr, n_cand, row_capacity, alpha * alpha, near, out,
                                       nout);
    GRAB_CHECK_LAUNCH();
  });
  GRAB_CUDA(cudaMemcpyAsync(n_accepted, nout, 4, cudaMemcpyDeviceToHost, st));
  GRAB_CUDA(cudaStreamSynchronize(st));
  GRAB_CUDA(cudaMemcpyAsync(out_accepted, out, *n_accepted * 8, cudaMemcpyDeviceToHost, st));
  GRAB_CUDA(cudaStreamSynchronize(st));
  cudaFree(dX);
}

void try_rewire_device(const float* X, uint64_t n_rows, uint32_t dim, uint32_t* row, uint32_t k_max, uint32_t v,
                       uint32_t q, double sq_dvq, double alpha, uint32_t k_local, int32_t* accepted,
                       int32_t* evicted_pos) {
  cudaStream_t st = 0;
  if (v >= n_rows || q >= n_rows) throw Error(GRAB_ERR_VALUE, "slot out of range");
  for (uint32_t j = 0; j < k_max; ++j)
    if (row[j] != kSentinel && row[j] >= n_rows) throw Error(GRAB_ERR_VALUE, "row entry out of range");
  const uint32_t dp = (dim + 3) / 4 * 4;
  float* dX = upload_rows(X, n_rows, dim, dp, st);
  Pool pool(st);
  uint32_t* drow = pool.alloc<uint32_t>(k_max);
  int32_t* res = pool.alloc<int32_t>(2);
  GRAB_CUDA(cudaMemcpyAsync(drow, row, k_max * 4, cudaMemcpyHostToDevice, st));
  by_nc(dp, [&](auto ncv) {
    constexpr int NC = decltype(ncv)::value;
    k_rewire_one<NC><<<1, 32, 0, st>>>(dX, dp, drow, k_max, v, q, sq_dvq, alpha * alpha, k_local, res);
    GRAB_CHECK_LAUNCH();
  });
  int32_t h[2];
  GRAB_CUDA(cudaMemcpyAsync(h, res, 8, cudaMemcpyDeviceToHost, st));
  GRAB_CUDA(cudaMemcpyAsync(row, drow, k_max * 4, cudaMemcpyDeviceToHost, st));
  GRAB_CUDA(cudaStreamSynchronize(st));
  cudaFree(dX);
  *accepted = h[0];
  *evicted_pos = h[1];
}

}  // namespace grab
