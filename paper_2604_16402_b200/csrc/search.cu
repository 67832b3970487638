// filtered_beam_search: Alg. 2 range-constrained beam search, one warp per query.
//
// Reference semantics restated (searcher.py):
//   seeds       _sample_seeds 101-153 (PCG64/Lemire draws, first-occurrence,
//               n_live and f32 range checks, ordered scan fallback lo,hi,lo+1..)
//   queue       CandidateQueue 52-82: (dist, slot) ascending, truncated to
//               itopk after every admit; frontier = first `width` unexpanded
//   loop        search 201-224: gather A rows, drop SENTINEL / slot >= n,
//               per-iteration unique, exact visited set (never re-admit),
//               scalar pre-check before any distance, stamp, admit
//   result      top_k + truncated flag 226-233
//
// B200 mapping (v2): a persistent grid of warps, each owning one query at a
// time, sized to fill every SM (>= 16 resident warps). Per-warp shared memory
// holds only the queue (single buffer, merged in place), the candidate buffer
// and the per-iteration dedup table (~7 KB at itopk 256). The exact visited set
// lives in a per-warp global table (L2-resident, cleared by the owning warp at
// query start) with CAS inserts issued for the whole iteration at once; a query
// whose inserts would pass 3/4 load is re-run with a worst-case table (never a
// forgetful hash, which would re-admit nodes and break parity). Each iteration
// issues all adjacency loads, then all Attr{scalar, slot} loads, then all
// visited CASes before consuming any, and candidate rows are fetched G at a
// time with 16-byte ld.global.nc; every distance is reduced in f64 with the
// library's one xor tree (bit-identical across kernels).
#include <cstdio>
#include <cstdlib>
#include <map>
#include <memory>
#include <algorithm>
#include <mutex>

#include "index.cuh"
#include "rng.cuh"
#include "search.cuh"

namespace grab {

__constant__ PcgJump c_jump;
__device__ __forceinline__ u128 jump_a(int j) { return ((u128)c_jump.a_hi[j] << 64) | c_jump.a_lo[j]; }
__device__ __forceinline__ u128 jump_g(int j) { return ((u128)c_jump.g_hi[j] << 64) | c_jump.g_lo[j]; }

void upload_pcg_jump_tables() {
  PcgJump t;
  u128 a = 1, g = 0;
  for (int j = 0; j <= 32; ++j) {
    t.a_lo[j] = (uint64_t)a;
    t.a_hi[j] = (uint64_t)(a >> 64);
    t.g_lo[j] = (uint64_t)g;
    t.g_hi[j] = (uint64_t)(g >> 64);
    g = g + a;  // G_{j+1} = G_j + MULT^j
    a = a * pcg_mult();
  }
  GRAB_CUDA(cudaMemcpyToSymbol(c_jump, &t, sizeof(t)));
}

__device__ __forceinline__ uint32_t hash32(uint32_t k) { return k * 0x9E3779B1u; }

// Visited-table accesses (global, per-warp, L2-resident). The tables are
// written (clears, atomics) and re-read throughout a query while the candidate
// row stream sweeps L2; with default priority their dirty lines were evicted and
// re-fetched mid-query (ncu: 1.31 GB of DRAM writes per cfg2 launch for a
// read-only search). Every table access therefore carries an L2 evict_last
// policy so the ~45 MB of live tables stay resident under the row stream
// (-DGRAB_VIS_NO_HINT restores plain accesses for A/B).
#ifndef GRAB_VIS_NO_HINT
// L2 policy of one query's table: evict_last for tables small enough that every
// resident warp's table fits the persisting set-aside (narrow ranges: 1 % and
// 10 % at 1M rows), evict_normal for wide ones (50 %: 222 MB of tables would
// only crowd the candidate rows out of L2)
__device__ __forceinline__ uint64_t vis_make_policy(bool persist) {
  uint64_t p;
  if (persist)
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  else
    asm("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint32_t vis_or(uint32_t* a, uint32_t v, uint64_t pol) {
  uint32_t o;
  asm volatile("atom.global.or.L2::cache_hint.b32 %0, [%1], %2, %3;" : "=r"(o) : "l"(a), "r"(v), "l"(pol) : "memory");
  return o;
}
// (ptxas rejects .L2::cache_hint on atom.cas: the hash mode's CAS is plain; its
// lines are kept hot by the hinted loads that probe them)
__device__ __forceinline__ uint32_t vis_cas(uint32_t* a, uint32_t cmp, uint32_t v) { return atomicCAS(a, cmp, v); }
__device__ __forceinline__ uint32_t vis_ld(const uint32_t* a, uint64_t pol) {
  uint32_t o;  // .cg: the L2 copy (the atomics live there), never a stale L1 line
  asm volatile("ld.global.cg.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(o) : "l"(a), "l"(pol) : "memory");
  return o;
}
__device__ __forceinline__ void vis_clear(uint32_t* p, uint32_t n, uint64_t pol) {
  for (uint32_t i = lane_id() * 4; i < n; i += 128)
    asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1, %1, %1, %1}, %2;" ::"l"(p + i), "r"(0u), "l"(pol)
                 : "memory");
}
#else
__device__ __forceinline__ uint64_t vis_make_policy(bool) { return 0; }
__device__ __forceinline__ uint32_t vis_or(uint32_t* a, uint32_t v, uint64_t) { return atomicOr(a, v); }
__device__ __forceinline__ uint32_t vis_cas(uint32_t* a, uint32_t cmp, uint32_t v) { return atomicCAS(a, cmp, v); }
__device__ __forceinline__ uint32_t vis_ld(const uint32_t* a, uint64_t) { return *((volatile const uint32_t*)a); }
__device__ __forceinline__ void vis_clear(uint32_t* p, uint32_t n, uint64_t) {
  const uint4 z = make_uint4(0, 0, 0, 0);
  for (uint32_t i = lane_id() * 4; i < n; i += 128) *reinterpret_cast<uint4*>(p + i) = z;
}
#endif
#ifndef GRAB_VIS_PERSIST_BYTES
#define GRAB_VIS_PERSIST_BYTES 16384u
#endif
// At query end a persisting table is dead (the next query clears it first):
// drop its lines from L2 without write-back, so persisting lines never linger
// into later launches (left in the set-aside they cost wide ranges a third of
// the L2 for normal lines: 20 % selectivity 5.8 -> 8.0 ms, measured).
__device__ __forceinline__ void vis_release(uint32_t* p, uint32_t n) {
  for (uint32_t i = lane_id() * 32; i < n; i += 32 * 32)
    asm volatile("discard.global.L2 [%0], 128;" ::"l"(p + i) : "memory");
}

// Open-addressing set of 2^lg u32 entries (value key+1, 0 = empty).
// Every probe loop is warp-uniform (all 32 lanes iterate until no lane has a
// pending probe): a per-lane trip count would leave the warp diverged, and a
// diverged warp runs every later shuffle/ballot through the slow collective
// path (BRA.DIV) -- measured at ~95% of all warp ops before this rule.
// Returns true for active lanes whose key was absent (and is now inserted).
__device__ __forceinline__ bool set_insert_w(uint32_t* tab, uint32_t lg, uint32_t key, bool active) {
  const uint32_t mask = (1u << lg) - 1;
  uint32_t h = hash32(key) >> (32 - lg);
  const uint32_t v = key + 1;
  uint32_t cur = active ? vis_cas(tab + h, 0u, v) : 0u;
  bool pending = active && cur != 0u && cur != v;
  while (__any_sync(0xFFFFFFFFu, pending)) {
    if (pending) {
      h = (h + 1) & mask;
      cur = vis_cas(tab + h, 0u, v);
      pending = cur != 0u && cur != v;
    }
  }
  return active && cur == 0u;
}

// True for active lanes whose key is present.
__device__ __forceinline__ bool set_contains_w(const uint32_t* tab, uint32_t lg, uint32_t key, bool active,
                                               uint64_t pol) {
  const uint32_t mask = (1u << lg) - 1;
  uint32_t h = hash32(key) >> (32 - lg);
  const uint32_t v = key + 1;
  uint32_t cur = active ? vis_ld(tab + h, pol) : 0u;
  bool pending = active && cur != 0u && cur != v;
  while (__any_sync(0xFFFFFFFFu, pending)) {
    if (pending) {
      h = (h + 1) & mask;
      cur = vis_ld(tab + h, pol);
      pending = cur != 0u && cur != v;
    }
  }
  return active && cur == v;
}

// Exact per-query visited set (searcher.py:90-98 epoch table). Only in-range
// nodes are ever stamped, and every in-range node lives in the slab interval
// [base, base + nbits) of the query's bucket interval, so when that interval
// fits the warp's table as a bitmap (<= 32 * 2^lg rows) the set is a bitmap:
// one atomicOr per insert, no probing, and only nbits/8 bytes to clear and to
// keep in L2. Wider intervals (e.g. full-range insert searches) use the
// open-addressing hash table.
struct Visited {
  uint32_t* tab;
  uint32_t lg, base, nbits;
  bool bm;
  uint64_t pol;  // L2 policy of this query's table accesses
  __device__ __forceinline__ uint32_t clear_words_n() const {
    return bm ? ((nbits + 4095u) >> 12) << 7 : (1u << lg);  // multiple of 128 words
  }
  __device__ __forceinline__ bool contains_w(uint32_t key, bool active) const {
    if (bm) {
      const uint32_t o = key - base;
      return active && (vis_ld(tab + (o >> 5), pol) >> (o & 31) & 1u);
    }
    return set_contains_w(tab, lg, key, active, pol);
  }
  __device__ __forceinline__ bool insert_w(uint32_t key, bool active) const {
    if (bm) {
      const uint32_t o = key - base;
      return active && !(vis_or(tab + (o >> 5), 1u << (o & 31), pol) >> (o & 31) & 1u);
    }
    return set_insert_w(tab, lg, key, active);
  }
};

__device__ __forceinline__ void clear_words(uint32_t* p, uint32_t n) {
  // n is a multiple of 128 (4 words per lane per step)
  const uint4 z = make_uint4(0, 0, 0, 0);
  for (uint32_t i = lane_id() * 4; i < n; i += 128) *reinterpret_cast<uint4*>(p + i) = z;
}

// ---------------------------------------------------------------- layout
__host__ __device__ inline uint32_t align16(uint32_t x) { return (x + 15u) & ~15u; }

// Per-warp shared memory. The queue is an array of 16-byte entries
// {f64 distance, slot, phys | kExpanded} kept sorted by (distance, slot), so a
// merge moves one LDS.128/STS.128 per displaced entry.
struct WarpLayout {
  uint32_t qe, cd, cs, cp, dd, fr, q, bytes;
};

__host__ __device__ inline WarpLayout warp_layout(const SearchShape& s) {
  WarpLayout l;
  uint32_t o = 0;
  l.qe = o;
  o += s.itopk * 16;
  l.cd = o;
  o += align16(s.cmax * 8);
  l.cs = o;
  o += align16(s.cmax * 4);
  l.cp = o;
  o += align16((s.cmax + 16) * 4);  // + a round of padding (pad_cands)
  l.dd = o;
  o += align16(s.dsz * 4);
  l.fr = o;
  o += align16(s.width * 4);
  l.q = o;  // query staging for wide rows (QueryRegs, NC >= 4)
  o += s.qbytes;
  l.bytes = o;
  return l;
}

constexpr uint32_t kExpanded = 0x80000000u;  // queue entry flag (phys ids < 2^31)
constexpr uint32_t kFull = 0xFFFFFFFFu;

__device__ __forceinline__ double qe_dist(const uint4& e) { return __hiloint2double((int)e.y, (int)e.x); }
__device__ __forceinline__ uint4 qe_pack(double d, uint32_t s, uint32_t p) {
  return make_uint4((uint32_t)__double2loint(d), (uint32_t)__double2hiint(d), s, p);
}

// ---------------------------------------------------------------- distances
// The query, one float4 per lane per 128-float chunk. Up to 2 chunks it lives
// in registers; wider rows (NC >= 4, e.g. d = 960) are staged in the warp's
// shared memory and read per chunk, so the row being scored keeps the
// registers (in registers the compiler also holds the f64 upcast: 16 regs/chunk).
template <int NC>
struct QueryRegs {
  static constexpr bool kShared = NC >= 4;
  float4 q[kShared ? 1 : NC];
  const float4* sq;
  __device__ __forceinline__ float4 get(int c) const { return kShared ? sq[c * 32 + lane_id()] : q[c]; }
};

template <int NC>
__device__ __forceinline__ void load_query(QueryRegs<NC>& r, const float* q, uint32_t dp, float4* stage) {
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const uint32_t col = (c * 32 + lane_id()) * 4;
    const float4 v = col < dp ? *reinterpret_cast<const float4*>(q + col) : make_float4(0, 0, 0, 0);
    if constexpr (QueryRegs<NC>::kShared)
      stage[c * 32 + lane_id()] = v;
    else
      r.q[c] = v;
  }
  r.sq = stage;
  __syncwarp();
}

template <int NC>
struct GroupOf {
#ifndef GRAB_SEARCH_G1
#define GRAB_SEARCH_G1 8
#endif
  static constexpr int G = NC == 1 ? GRAB_SEARCH_G1 : (NC == 2 ? 4 : (NC <= 4 ? 2 : 1));
};

// Distances for cand[0..n): writes cd[i]. All lanes participate; G rows are in
// flight per round (16-byte ld.global.nc per lane per 128-float chunk). The
// caller pads cp[n .. n+G) with a valid row id, so every round issues G
// unconditional loads (results past n are discarded). FULL: dp == 128*NC (no
// lane sits past the row end); otherwise every chunk load is predicated.
template <int NC, bool FULL>
__device__ __forceinline__ void score(const QueryRegs<NC>& qr, const float* __restrict__ X, uint32_t dp,
                                      const uint32_t* cp, double* cd, uint32_t n, bool deep_pf) {
  constexpr int G = GroupOf<NC>::G;
  const uint32_t lane = lane_id();
  const char* xl = reinterpret_cast<const char*>(X + lane * 4);  // this lane's first column
  const uint32_t rowb = dp * 4;
  // rolling L2 prefetch, PF rows ahead of the rows being loaded. Bitmap-mode
  // queries (the visited span fits the warp's table) prefetch ~4 KB (at least
  // one round of G): shallower is better once their tables stay in L2 (r02 A/B,
  // cfg2 10 %: 16 KB 3.78 ms, 8 KB 3.72, 4 KB 3.66, none 3.93; d = 960: 29.0 ->
  // 24.5 ms). Hash-mode queries (wide spans on large indexes: cfg5's 12.5M-row
  // shards) keep ~16 KB ahead: 130K -> 247K QPS there. Prefetched rows must stay
  // resident until used (a whole iteration at d = 960 overran L2).
#ifndef GRAB_PF_BYTES
#define GRAB_PF_BYTES 4096u
#endif
#ifndef GRAB_PF_BYTES_DEEP
#define GRAB_PF_BYTES_DEEP 16384u
#endif
  constexpr uint32_t PFS0 = GRAB_PF_BYTES / (NC * 512u), PFD0 = GRAB_PF_BYTES_DEEP / (NC * 512u);
  constexpr uint32_t PFS = PFS0 < (uint32_t)G ? (uint32_t)G : (PFS0 > 32u ? 32u : PFS0);
  constexpr uint32_t PFD = PFD0 < (uint32_t)G ? (uint32_t)G : (PFD0 > 32u ? 32u : PFD0);
  const uint32_t PF = deep_pf ? PFD : PFS;
#ifndef GRAB_NO_PF
  if (lane < PF && lane < n) {
    const float* r = X + (uint64_t)cp[lane] * dp;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(r), "r"(rowb) : "memory");
  }
#endif
  __syncwarp();
  for (uint32_t base = 0; base < n; base += G) {
#ifndef GRAB_NO_PF
    if (lane < (uint32_t)G && base + PF + lane < n) {
      const float* r = X + (uint64_t)cp[base + PF + lane] * dp;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(r), "r"(rowb) : "memory");
    }
#endif
    float4 x[G][NC];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const float* row = reinterpret_cast<const float*>(xl + (uint64_t)cp[base + g] * rowb);
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        if (FULL)
          x[g][c] = ldg_nc_f4(row + c * 128);
        else
          x[g][c] = (c * 32 + lane) * 4 < dp ? ldg_nc_f4(row + c * 128) : make_float4(0, 0, 0, 0);
      }
    }
    double part[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      double acc = 0.0;
#pragma unroll
      for (int c = 0; c < NC; ++c) acc = sq4(x[g][c], qr.get(c), acc);
      part[g] = acc;
    }
    const double v = reduce_scatter<G>(part);
    constexpr uint32_t SPAN = 32 / G;  // lanes holding each candidate's sum
    const uint32_t g = lane / SPAN;
    if ((lane % SPAN) == 0 && base + g < n) cd[base + g] = v;
  }
  __syncwarp();
}

// Pad cp[n .. n+16) with cp[0] so score() can issue whole rounds (G <= 16).
__device__ __forceinline__ void pad_cands(uint32_t* cp, uint32_t n) {
  __syncwarp();
  const uint32_t lane = lane_id();
  const uint32_t p0 = cp[0];
  if (lane < 16) cp[n + lane] = p0;
  __syncwarp();
}

// ---------------------------------------------------------------- queue ops
// Register bitonic sort of one (d, s, p) per lane, ascending across lanes
// [0, S) for S = 2^lgS (lanes >= S are sorted among themselves; callers put
// +inf pads there).
__device__ __forceinline__ void warp_sort(double& d, uint32_t& s, uint32_t& p, uint32_t lgS) {
  const uint32_t lane = lane_id();
  for (uint32_t k = 2; k <= (1u << lgS); k <<= 1) {
#pragma unroll 5
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      const double od = __shfl_xor_sync(kFull, d, j);
      const uint32_t os = __shfl_xor_sync(kFull, s, j);
      const uint32_t op = __shfl_xor_sync(kFull, p, j);
      const bool up = (lane & k) == 0;
      const bool lower = (lane & j) == 0;
      const bool olt = key_less(od, os, d, s);
      if ((lower == up) ? olt : !olt) {
        d = od;
        s = os;
        p = op;
      }
    }
  }
}

// Number of queue entries strictly less than (kd, ks): branch-free lower bound
// with a warp-uniform step count (no divergence).
__device__ __forceinline__ uint32_t rank_in_queue(const uint4* qe, uint32_t L, double kd, uint32_t ks) {
  uint32_t pos = 0;
  for (uint32_t step = L ? (1u << (31 - __clz(L))) : 0u; step > 0; step >>= 1) {
    const uint32_t probe = pos + step;
    if (probe <= L) {
      const double* qd = reinterpret_cast<const double*>(qe + probe - 1);
      const uint32_t qs = reinterpret_cast<const uint32_t*>(qe + probe - 1)[2];
      if (key_less(*qd, qs, kd, ks)) pos = probe;
    }
  }
  return pos;
}

// CandidateQueue.admit (searcher.py:64-71): merge the nc candidates (cd, cs,
// cp) into the queue of length L in place, truncated to itopk. Candidates that
// cannot beat the current tail are dropped first (compacted in place); the
// survivors are merged 32 at a time (chunk by chunk with truncation after each
// equals one merge of the union): sorted in registers (network sized to the
// chunk), each survivor's final position = its index + its rank in the queue
// (branch-free binary search), and every output position from the first new
// entry up is filled once, top chunk first, from either a survivor (shuffle)
// or the queue entry it displaces. `fu` (first-unexpanded hint) is lowered to
// the first new entry. Returns the new length.
__device__ __forceinline__ uint32_t admit(uint4* qe, double* cd, uint32_t* cs, uint32_t* cp, uint32_t L,
                                          uint32_t nc, uint32_t itopk, uint32_t& fu) {
  const uint32_t lane = lane_id();
  const double kInf = __longlong_as_double(0x7FF0000000000000ll);
  if (L == itopk && nc) {
    const uint4 te = qe[L - 1];
    const double td = qe_dist(te);
    uint32_t kept = 0;
    for (uint32_t b0 = 0; b0 < nc; b0 += 32) {
      const uint32_t i = b0 + lane;
      double d = 0;
      uint32_t s = 0, p = 0;
      bool ok = false;
      if (i < nc) {
        d = cd[i];
        s = cs[i];
        p = cp[i];
        ok = key_less(d, s, td, te.z);
      }
      const uint32_t m = __ballot_sync(kFull, ok);
      __syncwarp();
      if (ok) {
        const uint32_t pos = kept + __popc(m & ((1u << lane) - 1));
        cd[pos] = d;
        cs[pos] = s;
        cp[pos] = p;
      }
      kept += __popc(m);
    }
    __syncwarp();
    nc = kept;
  }
  for (uint32_t b0 = 0; b0 < nc; b0 += 32) {
    const uint32_t i = b0 + lane;
    double d = kInf;
    uint32_t s = kFull, p = kFull;
    bool ok = i < nc;
    if (ok) {
      d = cd[i];
      s = cs[i];
      p = cp[i];
    }
    if (b0 > 0 && L == itopk) {  // the tail moved since the prefilter
      const uint4 te = qe[L - 1];
      ok = ok && key_less(d, s, qe_dist(te), te.z);
    }
    const uint32_t cnt = __popc(__ballot_sync(kFull, ok));
    if (cnt == 0) continue;
    if (!ok) {
      d = kInf;
      s = kFull;
      p = kFull;
    }
    // survivors sit in lanes [0, navail): a network over the next power of 2 sorts them first
    const uint32_t navail = min(32u, nc - b0);
    warp_sort(d, s, p, navail <= 1 ? 0 : 32 - __clz(navail - 1));
    // final position of survivor i: i + (queue entries before it); distinct and increasing
    const uint32_t f = lane < cnt ? lane + rank_in_queue(qe, L, d, s) : kFull;
    const uint32_t f0 = __shfl_sync(kFull, f, 0);
    const uint32_t flast = __shfl_sync(kFull, f, cnt - 1);
    const uint32_t newL = min(itopk, L + cnt);
    // fill the output positions [f0, newL) chunk by chunk from the top: position
    // pos holds survivor (#survivors before pos) if some f == pos, else queue
    // entry pos - (#survivors before pos); every source index is <= pos, so
    // top-down chunks read their sources before anything below is written
    int32_t c0 = (int32_t)((newL - 1) & ~31u);
    // chunks above the last survivor are a plain shift by cnt (one LDS.128 +
    // STS.128 per entry): a chunk's reads [P0 - cnt, P0 + 31] never overlap the
    // writes of the chunks above it, so one __syncwarp (read before write inside
    // the chunk) is all the ordering it needs
    for (; c0 > (int32_t)flast; c0 -= 32) {
      const uint32_t pos = (uint32_t)c0 + lane;
      uint4 e = make_uint4(0, 0, 0, 0);
      if (pos < newL) e = qe[pos - cnt];
      __syncwarp();
      if (pos < newL) qe[pos] = e;
    }
    __syncwarp();
    for (; c0 >= (int32_t)(f0 & ~31u); c0 -= 32) {
      const uint32_t P0 = (uint32_t)c0, pos = P0 + lane;
      const uint32_t B = __reduce_or_sync(kFull, (f >= P0 && f < P0 + 32) ? 1u << (f - P0) : 0u);
      const uint32_t before = __popc(__ballot_sync(kFull, f < P0)) + __popc(B & ((1u << lane) - 1));
      const bool is_c = (B >> lane) & 1u;
      const double cdv = __shfl_sync(kFull, d, before & 31);
      const uint32_t csv = __shfl_sync(kFull, s, before & 31);
      const uint32_t cpv = __shfl_sync(kFull, p, before & 31);
      const bool live = pos >= f0 && pos < newL;
      uint4 e = make_uint4(0, 0, 0, 0);
      if (live && !is_c) e = qe[pos - before];
      __syncwarp();
      if (live) qe[pos] = is_c ? qe_pack(cdv, csv, cpv) : e;
      __syncwarp();
    }
    fu = min(fu, f0);
    L = newL;
  }
  return L;
}

// ---------------------------------------------------------------- seeds
// _sample_seeds (searcher.py:101-153). Draws of one jump-ahead round (64 words,
// lane L owns output 32r+L = words lo,hi) are compacted into `stage` in word
// order, then consumed 32 at a time in draw order. Returns seeds written to
// (cp, cs)[0..n); *attempts = SearchStats.seed_attempts.
__device__ uint32_t sample_seeds(const SearchArgs& a, uint32_t* stage, uint32_t* cp, uint32_t* cs, const Visited& vis,
                                 uint32_t lo_b, uint32_t hi_b, float lo_f, float hi_f,
                                 uint64_t rng_seed, uint32_t* attempts) {
  const uint32_t lane = lane_id();
  const uint32_t lt = (1u << lane) - 1;
  const uint32_t want = a.want;
  const uint64_t c0 = a.bcum[lo_b];
  const uint64_t total = a.bcum[hi_b + 1] - c0;
  uint32_t picked = 0;
  *attempts = 0;
  const uint32_t bstep = hi_b > lo_b ? 1u << (31 - __clz(hi_b - lo_b)) : 0u;
  if (total > 0) {
    const uint32_t ndraw = 4 * want;
    *attempts = ndraw;
    const uint32_t tot = (uint32_t)total;
    const uint32_t thresh = (0u - tot) % tot;
    const Pcg64 g = pcg64_from_seed(rng_seed);
    u128 st = jump_a(lane + 1) * g.state + g.inc * jump_g(lane + 1);
    const u128 a32 = jump_a(32), g32 = g.inc * jump_g(32);
    uint32_t drawn = 0;
    while (drawn < ndraw && picked < want) {
      uint32_t nround;
      if (tot == 1u) {  // numpy returns zeros without consuming words
        stage[lane] = 0;
        stage[lane + 32] = 0;
        nround = 64;
      } else {
        const uint64_t out = pcg_xsl_rr(st);
        st = a32 * st + g32;
        const uint64_t mlo = (uint64_t)(uint32_t)out * tot, mhi = (uint64_t)(uint32_t)(out >> 32) * tot;
        const bool alo = (uint32_t)mlo >= thresh, ahi = (uint32_t)mhi >= thresh;
        const uint32_t blo = __ballot_sync(0xFFFFFFFFu, alo), bhi = __ballot_sync(0xFFFFFFFFu, ahi);
        const uint32_t pre = __popc(blo & lt) + __popc(bhi & lt);
        if (alo) stage[pre] = (uint32_t)(mlo >> 32);
        if (ahi) stage[pre + (alo ? 1 : 0)] = (uint32_t)(mhi >> 32);
        nround = __popc(blo) + __popc(bhi);
      }
      __syncwarp();
      for (uint32_t off = 0; off < nround && drawn < ndraw && picked < want; off += 32) {
        const uint32_t navail = min(min(32u, nround - off), ndraw - drawn);
        const bool have = lane < navail;
        uint32_t phys = 0xFFFFFFFFu, slot = kNoSlot;
        float sv = 0.f;
        if (have) {
          const uint64_t f = c0 + stage[off + lane];
          uint32_t lo = lo_b;  // last bucket b in [lo_b, hi_b] with bcum[b] <= f (warp-uniform steps)
          for (uint32_t step = bstep; step > 0; step >>= 1)
            if (lo + step <= hi_b && __ldg(a.bcum + lo + step) <= f) lo += step;
          phys = __ldg(a.bstart + lo) + (uint32_t)(f - __ldg(a.bcum + lo));
          const Attr at = ld_attr(a.attr, phys);
          slot = at.slot;
          sv = at.s;
        }
        const bool inr = have && slot < a.n_live && sv >= lo_f && sv <= hi_f;
        const uint32_t same = __match_any_sync(0xFFFFFFFFu, inr ? phys : 0xFFFFFFFFu);
        const bool first = inr && (uint32_t)(__ffs(same) - 1) == lane;
        const bool seen = vis.contains_w(phys, first);  // every lane must call (warp-uniform loop)
        const bool fresh = first && !seen;
        const uint32_t fm = __ballot_sync(0xFFFFFFFFu, fresh);
        const uint32_t rank = __popc(fm & lt);
        const bool take = fresh && rank < want - picked;
        vis.insert_w(phys, take);
        if (take) {
          cp[picked + rank] = phys;
          cs[picked + rank] = slot;
        }
        picked += __popc(__ballot_sync(0xFFFFFFFFu, take));
        drawn += navail;
        __syncwarp();
      }
    }
  }
  if (picked < want) {
    // ordered scan fallback: buckets lo, hi, lo+1 .. hi-1 (searcher.py:140-152)
    const uint32_t nb = hi_b - lo_b + 1;
    for (uint32_t t = 0; t < nb && picked < want; ++t) {
      if (t == 1 && hi_b == lo_b) break;
      const uint32_t b = t == 0 ? lo_b : (t == 1 ? hi_b : lo_b + t - 1);
      const uint32_t s0 = __ldg(a.bstart + b), cnt = __ldg(a.bcount + b);
      for (uint32_t base = 0; base < cnt && picked < want; base += 32) {
        const uint32_t i = base + lane;
        bool ok = false;
        const uint32_t phys = s0 + i;
        uint32_t slot = 0;
        if (i < cnt) {
          const Attr at = ld_attr(a.attr, phys);
          slot = at.slot;
          ok = slot < a.n_live && at.s >= lo_f && at.s <= hi_f;
        }
        const bool seen = vis.contains_w(phys, ok);  // every lane must call (warp-uniform loop)
        ok = ok && !seen;
        const uint32_t msk = __ballot_sync(0xFFFFFFFFu, ok);
        const uint32_t rank = __popc(msk & lt);
        const bool take = ok && rank < want - picked;
        vis.insert_w(phys, take);
        if (take) {
          cp[picked + rank] = phys;
          cs[picked + rank] = slot;
        }
        picked += __popc(__ballot_sync(0xFFFFFFFFu, take));
        __syncwarp();
      }
    }
  }
  return picked;
}

// ---------------------------------------------------------------- phase profile
// -DGRAB_SEARCH_PROFILE: per-phase SM cycles summed over all warps (lab only;
// run_search prints the split after each launch). Phases: 0 query setup +
// seeds, 1 frontier, 2 adjacency gather + pre-check, 3 visited set,
// 4 compaction, 5 distances, 6 admit.
#ifdef GRAB_SEARCH_PROFILE
__device__ unsigned long long g_phase[8];
#define PROF_INIT() long long prof_t = clock64(); unsigned long long prof_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#define PROF(i) { const long long t_ = clock64(); prof_acc[i] += (unsigned long long)(t_ - prof_t); prof_t = t_; }
#define PROF_FLUSH() if (lane == 0) { for (int i_ = 0; i_ < 8; ++i_) atomicAdd(&g_phase[i_], prof_acc[i_]); }
#else
#define PROF_INIT()
#define PROF(i)
#define PROF_FLUSH()
#endif

// ---------------------------------------------------------------- kernel
// NC: 128-float chunks per row; EPL: gathered neighbours per lane per iteration
// (width * K_max <= 32 * EPL).
#ifndef GRAB_SEARCH_MINB
#define GRAB_SEARCH_MINB 6
#endif
// STATS: SearchStats requested (the per-iteration unique count is compiled in
// only then: its code costs the stats-free instance ~2 % even when skipped)
template <int NC, int EPL, bool FULL, bool STATS>
__global__ void __launch_bounds__(128, NC >= 16 ? 3 : (EPL >= 8 ? 4 : GRAB_SEARCH_MINB))
    k_search(SearchArgs a, SearchShape sh) {
  extern __shared__ __align__(16) uint8_t smem[];
  const uint32_t lane = lane_id();
  const uint32_t lt = (1u << lane) - 1;
  const uint32_t wib = threadIdx.x >> 5;
  const uint32_t wpb = blockDim.x >> 5;
  uint8_t* base = smem + wib * sh.warp_bytes;
  uint4* qe = (uint4*)(base + sh.o_qe);
  double* cd = (double*)(base + sh.o_cd);
  uint32_t* cs = (uint32_t*)(base + sh.o_cs);
  uint32_t* cp = (uint32_t*)(base + sh.o_cp);
  uint32_t* dd = (uint32_t*)(base + sh.o_dd);
  uint32_t* fr = (uint32_t*)(base + sh.o_fr);
  const uint32_t gw = blockIdx.x * wpb + wib;
  const uint32_t vlg = sh.vlog2;
  uint32_t* vtab = a.gtab + ((uint64_t)gw << vlg);
  const uint32_t vcap = (1u << vlg) / 4 * 3;
  const uint32_t nw = gridDim.x * wpb;
  const uint32_t dlg = 31 - __clz(sh.dsz);
  const uint32_t K = a.k_max;
  const uint32_t kshift = (K & (K - 1)) == 0 ? 31 - __clz(K) : 0;  // power-of-two K: shifts, not divisions
  const uint32_t nwork = a.nwork_dev ? *a.nwork_dev : a.nwork;

  auto next_item = [&](uint32_t cur) -> uint32_t {
    if (!a.work_ctr) return cur + nw;
    uint32_t it = 0;
    if (lane == 0) it = atomicAdd(a.work_ctr, 1u);
    return __shfl_sync(kFull, it, 0);
  };
  PROF_INIT()
  for (uint32_t item = a.work_ctr ? next_item(0) : gw; item < nwork; item = next_item(item)) {
    const uint32_t qi = a.qmap ? a.qmap[item] : item;
    const float lo_f = __double2float_rn(a.lower[(uint64_t)qi * a.range_stride]);
    const float hi_f = __double2float_rn(a.upper[(uint64_t)qi * a.range_stride]);
    uint32_t iterations = 0, expanded = 0, dist_evals = 0, seed_evals = 0, attempts = 0;
    uint32_t gath_l = 0, rej_l = 0;  // per-lane partial counts, summed at the end
    uint32_t L = 0;
    bool overflow = false;
    // !(lo <= hi) (inverted or NaN bounds reaching the kernel through the device
    // path): an empty result, never a wrapped bucket interval (lo_b > hi_b)
    if (a.n_live > 0 && a.m > 0 && lo_f <= hi_f) {
      QueryRegs<NC> qr;
      load_query<NC>(qr, a.qphys ? a.X + (uint64_t)a.qphys[qi] * a.dp : a.Q + (uint64_t)qi * a.dp, a.dp,
                     (float4*)(base + sh.o_q));
      const uint32_t lo_b = bucket_of_f32(a.bound, a.m, lo_f);
      const uint32_t hi_b = bucket_of_f32(a.bound, a.m, hi_f);
      Visited vis;
      vis.tab = vtab;
      vis.lg = vlg;
      vis.base = __ldg(a.bstart + lo_b);
      vis.nbits = __ldg(a.bstart + hi_b) + __ldg(a.bcount + hi_b) - vis.base;
      vis.bm = vis.nbits <= (32u << vlg);
      vis.pol = vis_make_policy(vis.clear_words_n() * 4u <= GRAB_VIS_PERSIST_BYTES);
      vis_clear(vtab, vis.clear_words_n(), vis.pol);
      __syncwarp();
      const uint64_t seed = a.seeds ? a.seeds[qi] : derive_query_seed(a.seed_base, a.ordinal0 + qi);
      const uint32_t ns = sample_seeds(a, dd, cp, cs, vis, lo_b, hi_b, lo_f, hi_f, seed, &attempts);
      __syncwarp();
      clear_words(dd, sh.dsz);  // (the seed stage used it) all-zero from here on
      __syncwarp();
      uint32_t vis_n = ns;
      uint32_t fu = 0;  // every queue entry before fu is expanded
      if (ns > 0) {
        pad_cands(cp, ns);
        score<NC, FULL>(qr, a.X, a.dp, cp, cd, ns, !vis.bm);
        dist_evals = seed_evals = ns;
        L = admit(qe, cd, cs, cp, 0, ns, sh.itopk, fu);
        PROF(0)
        for (uint32_t it = 0; it < a.max_iter; ++it) {
          // frontier: first `width` unexpanded entries (searcher.py:73-79)
          uint32_t nf = 0;
          for (uint32_t b0 = fu & ~31u; b0 < L && nf < sh.width; b0 += 32) {
            const uint32_t i = b0 + lane;
            uint32_t w = 0;
            bool un = false;
            if (i < L && i >= fu) {
              w = qe[i].w;
              un = (w & kExpanded) == 0;
            }
            const uint32_t m = __ballot_sync(kFull, un);
            const uint32_t rank = __popc(m & lt);
            const bool pick = un && nf + rank < sh.width;
            if (pick) {
              fr[nf + rank] = w;
              qe[i].w = w | kExpanded;
            }
            const uint32_t pm = __ballot_sync(kFull, pick);
            if (pm) fu = b0 + 32 - __clz(pm);  // one past the last picked entry
            nf += __popc(pm);
          }
          __syncwarp();
          PROF(1)
          if (nf == 0) break;
          const uint32_t fan = nf * K;
          if (!vis.bm && vis_n + fan > vcap) {  // (a bitmap cannot overflow)
            overflow = true;
            break;
          }
          iterations++;
          expanded += nf;
          // (1) adjacency entries of the frontier rows + their {scalar, slot}
          uint32_t v[EPL];
          uint2 at[EPL];
#pragma unroll
          for (int t = 0; t < EPL; ++t) {
            const uint32_t e = lane + 32 * t;
            v[t] = kSentinel;
            at[t] = make_uint2(0x7FC00000u, kNoSlot);
            if (e < fan) {
              const uint32_t row = kshift ? e >> kshift : e / K;  // K = 32: row t, column lane
              const uint64_t idx = (uint64_t)fr[row] * K + (e - row * K);
              v[t] = __ldg(a.adj + idx);
              at[t] = __ldg(reinterpret_cast<const uint2*>(a.adja) + idx);
            }
          }
          __syncwarp();
          // (2) drop SENTINEL / slot >= n, scalar pre-check. Duplicates of an
          // in-range id are admitted once by the visited set below; the
          // per-iteration unique (np.unique, searcher.py:212) only feeds the
          // `gathered` / `precheck_rejected` counters, so it runs beside the
          // visited atomics (count_unique) instead of in front of them
          uint32_t cand_bits = 0;
#pragma unroll
          for (int t = 0; t < EPL; ++t) {
            const float sv = __uint_as_float(at[t].x);
            cand_bits |= (at[t].y < a.n_live && sv >= lo_f && sv <= hi_f) ? 1u << t : 0u;
          }
          PROF(2)
          // every first-probe CAS in flight before any is consumed; the table
          // (load <= 1/4) is left all-zero again by undoing this iteration's inserts
          auto count_unique = [&]() {
            const uint32_t dmask = (1u << dlg) - 1;
            uint32_t hs[EPL], dc[EPL], act = 0, pend = 0;
#pragma unroll
            for (int t = 0; t < EPL; ++t) {
              act |= at[t].y < a.n_live ? 1u << t : 0u;
              hs[t] = hash32(v[t]) >> (32 - dlg);
              dc[t] = ((act >> t) & 1u) ? atomicCAS(dd + hs[t], 0u, v[t] + 1) : 0u;
            }
#pragma unroll
            for (int t = 0; t < EPL; ++t) pend |= (((act >> t) & 1u) && dc[t] != 0u && dc[t] != v[t] + 1) ? 1u << t : 0u;
            while (__any_sync(kFull, pend != 0u)) {
#pragma unroll
              for (int t = 0; t < EPL; ++t) {
                if ((pend >> t) & 1u) {
                  hs[t] = (hs[t] + 1) & dmask;
                  dc[t] = atomicCAS(dd + hs[t], 0u, v[t] + 1);
                  if (dc[t] == 0u || dc[t] == v[t] + 1) pend &= ~(1u << t);
                }
              }
            }
            __syncwarp();
#pragma unroll
            for (int t = 0; t < EPL; ++t) {
              const bool uq = ((act >> t) & 1u) && dc[t] == 0u;
              if (uq) dd[hs[t]] = 0u;
              const float sv = __uint_as_float(at[t].x);
              gath_l += uq;
              rej_l += uq && !(sv >= lo_f && sv <= hi_f);
            }
            __syncwarp();
          };
          // (3) exact visited set: every first-probe atomic of the iteration in flight at once
          {
            uint32_t cur[EPL];
            if (vis.bm) {
#pragma unroll
              for (int t = 0; t < EPL; ++t) {
                const uint32_t o = v[t] - vis.base;
                cur[t] = ((cand_bits >> t) & 1u) ? vis_or(vtab + (o >> 5), 1u << (o & 31), vis.pol) : 0u;
              }
              if constexpr (STATS) count_unique();  // overlaps the visited atomics' round trip
#pragma unroll
              for (int t = 0; t < EPL; ++t)
                if ((cur[t] >> ((v[t] - vis.base) & 31)) & 1u) cand_bits &= ~(1u << t);
            } else {
              if constexpr (STATS) count_unique();
              const uint32_t vmask = (1u << vlg) - 1;
              uint32_t h[EPL];
#pragma unroll
              for (int t = 0; t < EPL; ++t) {
                h[t] = hash32(v[t]) >> (32 - vlg);
                cur[t] = ((cand_bits >> t) & 1u) ? vis_cas(vtab + h[t], 0u, v[t] + 1) : 0u;
              }
              uint32_t pend = 0;  // rare collisions: probe on, warp-uniformly
#pragma unroll
              for (int t = 0; t < EPL; ++t)
                pend |= (((cand_bits >> t) & 1u) && cur[t] != 0u && cur[t] != v[t] + 1) ? 1u << t : 0u;
              while (__any_sync(kFull, pend != 0u)) {
#pragma unroll
                for (int t = 0; t < EPL; ++t) {
                  if ((pend >> t) & 1u) {
                    h[t] = (h[t] + 1) & vmask;
                    cur[t] = vis_cas(vtab + h[t], 0u, v[t] + 1);
                    if (cur[t] == 0u || cur[t] == v[t] + 1) pend &= ~(1u << t);
                  }
                }
              }
#pragma unroll
              for (int t = 0; t < EPL; ++t)
                if (cur[t] != 0u) cand_bits &= ~(1u << t);
            }
          }
          __syncwarp();
          PROF(3)
          // (4) compact candidates in gather order
          uint32_t nc = 0;
#pragma unroll
          for (int t = 0; t < EPL; ++t) {
            const bool c = (cand_bits >> t) & 1u;
            const uint32_t cm = __ballot_sync(kFull, c);
            if (c) {
              const uint32_t pos = nc + __popc(cm & lt);
              cp[pos] = v[t];
              cs[pos] = at[t].y;
            }
            nc += __popc(cm);
          }
          __syncwarp();
          vis_n += nc;
          PROF(4)
          if (nc == 0) continue;
          dist_evals += nc;
          pad_cands(cp, nc);
          score<NC, FULL>(qr, a.X, a.dp, cp, cd, nc, !vis.bm);
          PROF(5)
          L = admit(qe, cd, cs, cp, L, nc, sh.itopk, fu);
          PROF(6)
        }
      }
      if (vis.clear_words_n() * 4u <= GRAB_VIS_PERSIST_BYTES) {
        __syncwarp();  // every lane's table accesses are done
        vis_release(vtab, vis.clear_words_n());
      }
    }
    if (overflow) {
      if (lane == 0 && a.ovf_count) {
        const uint32_t pos = atomicAdd(a.ovf_count, 1u);
        a.ovf_list[pos] = qi;
      }
      __syncwarp();
      continue;
    }
    const uint32_t cnt = min(L, a.k);
    for (uint32_t i = lane; i < a.k; i += 32) {
      int64_t s = -1;
      double d = __longlong_as_double(0x7FF8000000000000ll);
      if (i < cnt) {
        const uint4 e = qe[i];
        s = (int64_t)e.z;
        d = qe_dist(e);
      }
      a.out_slots[(uint64_t)qi * a.k + i] = s;
      a.out_dists[(uint64_t)qi * a.k + i] = d;
    }
    if constexpr (STATS) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        gath_l += __shfl_xor_sync(kFull, gath_l, o);
        rej_l += __shfl_xor_sync(kFull, rej_l, o);
      }
    }
    if (lane == 0) {
      a.out_counts[qi] = cnt;
      if (STATS && a.out_stats) {
        grab_search_stats st;
        st.iterations = iterations;
        st.dist_evals = dist_evals;
        st.seed_evals = seed_evals;
        st.gathered = gath_l;
        st.in_range_new = dist_evals - seed_evals;
        st.precheck_rejected = rej_l;
        st.seed_attempts = attempts;
        st.expanded = expanded;
        a.out_stats[qi] = st;
      }
    }
    __syncwarp();
    PROF(7)
  }
  PROF_FLUSH()
}

// adja[i] = attr[adj[i]] ({NaN, kNoSlot} for SENTINEL)
__global__ void k_fill_adja(const uint32_t* __restrict__ adj, const Attr* __restrict__ attr, uint64_t n,
                            uint2* __restrict__ out) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t v = adj[i];
  out[i] = v == kSentinel ? make_uint2(0x7FC00000u, kNoSlot) : __ldg(reinterpret_cast<const uint2*>(attr) + v);
}

void ensure_adja(const DevIndex& ix, cudaStream_t st) {
  DevIndex::AdjaSync& sy = *ix.adja_sync;
  std::lock_guard<std::mutex> lk(sy.mu);
  if (ix.adja && ix.adja_rows == ix.phys_cap && ix.adja_version == ix.adj_version) {
    if (sy.ready) GRAB_CUDA(cudaStreamWaitEvent(st, sy.ready, 0));  // (free once the fill has run)
    return;
  }
  const uint64_t n = ix.phys_cap * ix.params.k_max;
  if (!ix.adja || ix.adja_rows != ix.phys_cap) {
    if (ix.adja) {
      GRAB_CUDA(cudaStreamSynchronize(st));
      cudaFree(ix.adja);
      ix.adja = nullptr;
    }
    GRAB_CUDA(cudaMalloc(&ix.adja, std::max<uint64_t>(n, 1) * sizeof(Attr)));
    ix.adja_rows = ix.phys_cap;
  }
  if (n) {
    k_fill_adja<<<(unsigned)div_up(n, 256), 256, 0, st>>>(ix.adj, ix.attr, n, reinterpret_cast<uint2*>(ix.adja));
    GRAB_CHECK_LAUNCH();
  }
  ix.adja_version = ix.adj_version;
  if (!sy.ready) GRAB_CUDA(cudaEventCreateWithFlags(&sy.ready, cudaEventDisableTiming));
  GRAB_CUDA(cudaEventRecord(sy.ready, st));
}

// ---------------------------------------------------------------- host
static uint32_t ceil_log2(uint64_t x) {
  uint32_t l = 0;
  while ((1ull << l) < x) ++l;
  return l;
}

SearchShape make_shape(uint32_t itopk, uint32_t width, uint32_t k_max, uint32_t want, uint32_t max_iter, bool worst,
                       uint32_t dp, uint64_t live_rows, bool stats, uint64_t phys_rows) {
  SearchShape s;
  const uint32_t nc = (dp + 127) / 128;
  s.qbytes = nc > 2 ? (nc <= 4 ? 4u : nc <= 8 ? 8u : 16u) * 512u : 0u;  // QueryRegs<NC>::kShared staging
  s.itopk = itopk;
  s.width = width;
  const uint32_t fan = width * k_max;
  s.cmax = 1u << ceil_log2(std::max<uint64_t>(std::max(fan, want), 32));  // bitonic pads to a power of 2
  // dedup table, load <= 1/4; it only exists for the SearchStats counters: the
  // stats-free instance keeps just the 64-word seed stage that shares it (2 KB
  // less shared memory per warp at width 4: 5 -> 6 blocks per SM at itopk 400)
  s.dsz = stats ? 1u << ceil_log2(std::max<uint64_t>(4ull * fan, 128)) : 64u;
  if (!worst) {
    // sized for the visits of a wide (hash-mode) search: ~itopk * 36 at full range (1M rows, itopk 128:
    // a 4K table overflowed every insert candidate search); a bitmap needs only nbits / 8 of it
    s.vlog2 = std::min<uint32_t>(15, std::max<uint32_t>(12, ceil_log2((uint64_t)itopk * 48)));
    // when every query's slab interval fits, size the table as a bitmap over all
    // phys rows (<= 2^17 words = 512 KB per warp, i.e. indexes up to 4M rows):
    // full-range searches (the insert's candidate search) then use one atomicOr
    // per candidate instead of CAS probe chains (measured: 53.8 -> 48.3 ms per
    // 100K candidate searches at 1M rows). Only an interval's own words are
    // ever cleared, so narrow searches pay nothing for the larger allocation.
    // (GRAB_SEARCH_HASH_VISITED=1 keeps the itopk-sized table, i.e. the hash
    // path, for wide spans: what indexes above 4M rows always run; tests use it)
    const uint32_t need = ceil_log2(std::max<uint64_t>(1, (phys_rows + 31) / 32));
    if (need <= 17 && !getenv("GRAB_SEARCH_HASH_VISITED")) s.vlog2 = std::max(s.vlog2, need);
    if (const char* e = getenv("GRAB_SEARCH_VLOG2")) s.vlog2 = (uint32_t)atoi(e);  // (lab knob)
  } else {
    // every insert is a distinct in-range row, so the live row count bounds the
    // table too (max_iterations is only a cap: 1e6 must not size a 5 GB table)
    const uint64_t bound = std::min<uint64_t>((uint64_t)want + (uint64_t)max_iter * fan + fan,
                                              (uint64_t)live_rows + fan);
    s.vlog2 = std::max<uint32_t>(11, ceil_log2(bound * 4 / 3 + 1));
  }
  const WarpLayout l = warp_layout(s);
  s.o_qe = l.qe;
  s.o_cd = l.cd;
  s.o_cs = l.cs;
  s.o_cp = l.cp;
  s.o_dd = l.dd;
  s.o_fr = l.fr;
  s.o_q = l.q;
  s.warp_bytes = l.bytes;
  return s;
}

// Calls f(kernel) with the k_search instance for (nc, epl, full, stats).
template <typename F>
static void with_kernel(uint32_t nc, uint32_t epl, bool full, bool stats, F&& f) {
#define GRAB_K(NC_, EPL_)                                         \
  if (nc == NC_ && epl == EPL_) {                                 \
    if (full)                                                     \
      stats ? f(k_search<NC_, EPL_, true, true>) : f(k_search<NC_, EPL_, true, false>);   \
    else                                                          \
      stats ? f(k_search<NC_, EPL_, false, true>) : f(k_search<NC_, EPL_, false, false>); \
    return;                                                       \
  }
  GRAB_K(1, 1) GRAB_K(1, 2) GRAB_K(1, 4) GRAB_K(2, 1) GRAB_K(2, 2) GRAB_K(2, 4)
  GRAB_K(4, 1) GRAB_K(4, 2) GRAB_K(4, 4) GRAB_K(8, 1) GRAB_K(8, 2) GRAB_K(8, 4)
  GRAB_K(1, 8) GRAB_K(2, 8) GRAB_K(4, 8) GRAB_K(8, 8)  // width * K_max up to 256 (e.g. K_max 64, width 4)
  GRAB_K(16, 1) GRAB_K(16, 2) GRAB_K(16, 4) GRAB_K(16, 8)  // 1024 < d <= 2048
#undef GRAB_K
  throw Error(GRAB_ERR_VALUE, "unsupported search kernel shape");
}

// Launches one search grid: min(work, resident capacity) blocks of 4 warps,
// `max_blocks` caps the grid (worst-case retry: bounded table memory).
static void launch(SearchArgs a, const SearchShape& sh, int num_sms, cudaStream_t st, DBufLite& tables,
                   uint64_t max_blocks) {
  const WarpLayout lay = warp_layout(sh);
  const uint32_t wpb = 4;
  const uint32_t smem = lay.bytes * wpb;
  if (smem > 227 * 1024) throw Error(GRAB_ERR_VALUE, "search parameters exceed shared memory (itopk too large)");
  uint32_t nc = (uint32_t)div_up(a.dp, 128);
  nc = nc <= 1 ? 1 : nc <= 2 ? 2 : nc <= 4 ? 4 : nc <= 8 ? 8 : nc <= 16 ? 16 : 0;
  if (!nc) throw Error(GRAB_ERR_VALUE, "dimension > 2048 not supported by the search kernel");
  uint32_t epl = (uint32_t)div_up(sh.width * a.k_max, 32);
  epl = epl <= 1 ? 1 : epl <= 2 ? 2 : epl <= 4 ? 4 : 8;
  if (epl > 8 || sh.cmax > 256) throw Error(GRAB_ERR_VALUE, "search_width * k_max > 256 not supported");
  const bool full = a.dp == nc * 128;
  // launch configuration per (instance, smem): the attribute / occupancy calls
  // cost tens of microseconds, so they run once per configuration and device
  int dev = 0;
  GRAB_CUDA(cudaGetDevice(&dev));
  const bool stats = a.out_stats != nullptr;
  const uint64_t key = ((uint64_t)dev << 48) | ((uint64_t)nc << 40) | ((uint64_t)epl << 36) |
                       ((uint64_t)full << 35) | ((uint64_t)stats << 34) | smem;
  static std::mutex occ_mu;
  static std::map<uint64_t, int> occ;
  int per_sm = 0;
  {
    std::lock_guard<std::mutex> g(occ_mu);
    auto it = occ.find(key);
    if (it != occ.end()) {
      per_sm = it->second;
    } else {
      with_kernel(nc, epl, full, stats, [&](auto kern) {
        // the attribute is per kernel instance: always the device maximum, so a
        // later, smaller configuration never lowers it under a cached larger one
        GRAB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        GRAB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        GRAB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * wpb, smem));
      });
      per_sm = std::max(per_sm, 1);
      occ[key] = per_sm;
    }
  }
  uint64_t cap_blocks = (uint64_t)per_sm * num_sms;
  if (const char* e = getenv("GRAB_SEARCH_BLOCKS")) cap_blocks = std::min<uint64_t>(cap_blocks, strtoull(e, 0, 10));
  const uint64_t blocks = std::min<uint64_t>(std::min<uint64_t>(div_up(a.nwork, wpb), cap_blocks), max_blocks);
  if (!blocks) return;
  // one visited table per resident warp
  const uint64_t words = blocks * wpb * (1ull << sh.vlog2);
  tables.ensure(words * 4, st);
  a.gtab = (uint32_t*)tables.p;
  with_kernel(nc, epl, full, stats, [&](auto kern) {
    kern<<<(uint32_t)blocks, 32 * wpb, smem, st>>>(a, sh);
    GRAB_CHECK_LAUNCH();
  });
}

// Stream-ordered and host-sync free: queries whose visited table would pass
// 3/4 load are listed by the main grid and re-run exactly by a second grid with
// a worst-case table; that grid reads its work count on the device (and exits
// at once when nothing overflowed).
// Scratch of one stream: reused by every later search on that stream (stream
// order makes the reuse safe without host synchronization).
struct SearchWs {
  std::mutex mu;  // host-side: one enqueue at a time per stream (threads may share a stream)
  DBufLite tables, big_tables, ovf, ctr, order;
};
struct SearchWsCache {
  std::mutex mu;
  std::map<cudaStream_t, std::unique_ptr<SearchWs>> by_stream;
};

void free_search_ws(DevIndex& ix) {
  if (!ix.search_ws) return;
  cudaDeviceSynchronize();
  ix.search_ws->by_stream.clear();  // DBufLite frees stream-ordered
  cudaDeviceSynchronize();
  ix.search_ws.reset();
}

static SearchWs& workspace(const DevIndex& ix, cudaStream_t st) {
  static std::mutex init_mu;
  {
    std::lock_guard<std::mutex> g(init_mu);
    if (!ix.search_ws) const_cast<DevIndex&>(ix).search_ws = std::make_shared<SearchWsCache>();
  }
  SearchWsCache& c = *ix.search_ws;
  std::lock_guard<std::mutex> g(c.mu);
  auto& slot = c.by_stream[st];
  if (!slot) slot = std::make_unique<SearchWs>();
  return *slot;
}

// L2 set-aside for persisting lines. Narrow-range queries keep their visited
// table (<= 16 KB) in L2 with evict_last accesses, and those stay resident only
// inside the persisting set-aside. A fixed 48 MB set-aside, reserved once per
// device, is the measured balance (r02, cfg2; ms per 10K queries at 0 / 32 /
// 48 / 64 MB): 10 %: 3.94 / 3.78 / 3.70 / 3.66; 5 %: 2.78 / 2.62 / 2.59 / 2.59;
// 20 %: 5.76 / 5.75 / 5.82 / 6.85; 50 %: 10.0 / 10.0 / 10.2 / 12.6. (Switching
// the set-aside per launch from the batch's table sizes was tried: reconfiguring
// it while kernels run stalled a launch by 22 ms.) GRAB_L2_PERSIST_MB overrides
// the size (0 = none).
static void reserve_persisting_l2() {
  static std::mutex mu;
  static std::vector<int> done;
  int dev = 0;
  GRAB_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> g(mu);
  if (std::find(done.begin(), done.end(), dev) != done.end()) return;
  done.push_back(dev);
  size_t want = (size_t)48 << 20;
  if (const char* e = getenv("GRAB_L2_PERSIST_MB")) want = (size_t)atoi(e) << 20;
  int mx = 0;
  if (cudaDeviceGetAttribute(&mx, cudaDevAttrMaxPersistingL2CacheSize, dev) != cudaSuccess || mx <= 0) {
    cudaGetLastError();
    return;
  }
  cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, std::min(want, (size_t)mx));
  cudaGetLastError();  // best effort: never fail a search over the cache reservation
}

// Work order of a batch with per-query ranges: queries claimed in the order of
// their lower bound, so the warps resident at any moment search overlapping
// slab spans and share the rows they read in L2 (random order spreads the
// resident queries over the whole index). Results are written at the query's
// own index and every query's search is independent of the order.
// One block: 2048 bins over [min, max] of the finite lower bounds (unbounded
// ones go to the end bins), counting sort, order inside a bin arbitrary.
constexpr uint32_t kOrderBins = 2048, kOrderThreads = 1024;

// `lower` may be page-locked host memory (the zero-copy path): it is read
// once, 8 loads in flight per thread, into the device copy `lf` that the
// histogram and scatter passes use.
__global__ void __launch_bounds__(kOrderThreads) k_order_by_lower(const double* lower, uint64_t stride, uint32_t n,
                                                                  float* lf, uint32_t* order) {
  __shared__ uint32_t cnt[kOrderBins];
  __shared__ float wmin[32], wmax[32];
  const uint32_t t = threadIdx.x, lane = t & 31, w = t >> 5;
  float mn = INFINITY, mx = -INFINITY;
  constexpr uint32_t B = 8;
  for (uint32_t i0 = t; i0 < n; i0 += B * kOrderThreads) {
    double x[B];
#pragma unroll
    for (uint32_t b = 0; b < B; ++b) {
      const uint32_t i = i0 + b * kOrderThreads;
      x[b] = i < n ? lower[(uint64_t)i * stride] : 0.0;
    }
#pragma unroll
    for (uint32_t b = 0; b < B; ++b) {
      const uint32_t i = i0 + b * kOrderThreads;
      if (i >= n) break;
      const float v = __double2float_rn(x[b]);
      lf[i] = v;
      if (isfinite(v)) {
        mn = fminf(mn, v);
        mx = fmaxf(mx, v);
      }
    }
  }
  for (uint32_t o = 16; o; o >>= 1) {
    mn = fminf(mn, __shfl_xor_sync(0xFFFFFFFFu, mn, o));
    mx = fmaxf(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
  }
  if (lane == 0) {
    wmin[w] = mn;
    wmax[w] = mx;
  }
  for (uint32_t b = t; b < kOrderBins; b += kOrderThreads) cnt[b] = 0;
  __syncthreads();
  mn = wmin[lane];
  mx = wmax[lane];
  for (uint32_t o = 16; o; o >>= 1) {
    mn = fminf(mn, __shfl_xor_sync(0xFFFFFFFFu, mn, o));
    mx = fmaxf(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
  }
  const float scale = mx > mn ? (float)(kOrderBins - 1) / (mx - mn) : 0.f;
  auto bin_of = [&](uint32_t i) -> uint32_t {
    const float v = lf[i];  // written by this thread in the first pass (same i -> same thread)
    if (!(v >= mn)) return 0;  // -inf (and NaN: any bin is fine)
    if (!(v <= mx)) return kOrderBins - 1;
    return min(kOrderBins - 1, (uint32_t)((v - mn) * scale));
  };
  for (uint32_t i = t; i < n; i += kOrderThreads) atomicAdd(&cnt[bin_of(i)], 1u);
  __syncthreads();
  if (w == 0) {  // exclusive scan of the bins by one warp (64 bins per lane)
    constexpr uint32_t per = kOrderBins / 32;
    uint32_t sum = 0;
    for (uint32_t j = 0; j < per; ++j) sum += cnt[lane * per + j];
    uint32_t inc = sum;
    for (uint32_t o = 1; o < 32; o <<= 1) {
      const uint32_t x = __shfl_up_sync(0xFFFFFFFFu, inc, o);
      if (lane >= o) inc += x;
    }
    uint32_t run = inc - sum;
    for (uint32_t j = 0; j < per; ++j) {
      const uint32_t c = cnt[lane * per + j];
      cnt[lane * per + j] = run;
      run += c;
    }
  }
  __syncthreads();
  for (uint32_t i = t; i < n; i += kOrderThreads) order[atomicAdd(&cnt[bin_of(i)], 1u)] = i;
}

constexpr uint32_t kOrderMinQueries = 2048;  // smaller batches fit in one wave of resident warps

// Work order of a batch with ONE shared range (search_batch, the insert's
// full-range candidate search): queries grouped by where they lie in vector
// space, so resident warps walk overlapping graph neighbourhoods and share the
// rows they read in L2. Cell = signs of kSimBits random +-1 projections, each
// taken relative to the batch mean of that projection; cells sorted as integers
// (the first projections are the coarsest split).
constexpr uint32_t kSimBits = 10;

__device__ __forceinline__ uint32_t sim_hash(uint32_t x) {  // lowbias32
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}

// warp per query: proj[q][j] = sum_c x[c] * (+-1), sign bit `lane` of hash(j, c / 32)
__global__ void k_sim_project(const float* Q, const uint32_t* qphys, const float* X, uint32_t dp, uint32_t n,
                              float* proj, float* sums) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t w0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  float tot[kSimBits];
#pragma unroll
  for (uint32_t j = 0; j < kSimBits; ++j) tot[j] = 0.f;
  for (uint32_t q = w0; q < n; q += nw) {
    const float* row = qphys ? X + (uint64_t)qphys[q] * dp : Q + (uint64_t)q * dp;
    float acc[kSimBits];
#pragma unroll
    for (uint32_t j = 0; j < kSimBits; ++j) acc[j] = 0.f;
    for (uint32_t c = lane, i = 0; c < dp; c += 32, ++i) {
      const float x = __ldg(row + c);
#pragma unroll
      for (uint32_t j = 0; j < kSimBits; ++j)
        acc[j] += ((sim_hash(j * 4096u + i) >> lane) & 1u) ? x : -x;
    }
#pragma unroll
    for (uint32_t j = 0; j < kSimBits; ++j) {
      float v = acc[j];
      for (uint32_t o = 16; o; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
      acc[j] = v;
      tot[j] += v;
    }
    if (lane < kSimBits) {
      float mine = acc[0];
#pragma unroll
      for (uint32_t j = 1; j < kSimBits; ++j) mine = lane == j ? acc[j] : mine;
      proj[(uint64_t)q * kSimBits + lane] = mine;
    }
  }
  if (lane == 0) {
#pragma unroll
    for (uint32_t j = 0; j < kSimBits; ++j) atomicAdd(&sums[j], tot[j]);
  }
}

// one block: counting sort of the queries by cell
__global__ void __launch_bounds__(kOrderThreads) k_order_by_cell(const float* proj, const float* sums, uint32_t n,
                                                                 uint32_t* order) {
  constexpr uint32_t NB = 1u << kSimBits;
  __shared__ uint32_t cnt[NB];
  __shared__ float mean[kSimBits];
  const uint32_t t = threadIdx.x, lane = t & 31, w = t >> 5;
  if (t < kSimBits) mean[t] = sums[t] / (float)n;
  for (uint32_t b = t; b < NB; b += kOrderThreads) cnt[b] = 0;
  __syncthreads();
  auto cell = [&](uint32_t q) -> uint32_t {
    uint32_t c = 0;
#pragma unroll
    for (uint32_t j = 0; j < kSimBits; ++j) c = (c << 1) | (proj[(uint64_t)q * kSimBits + j] > mean[j] ? 1u : 0u);
    return c;
  };
  for (uint32_t q = t; q < n; q += kOrderThreads) atomicAdd(&cnt[cell(q)], 1u);
  __syncthreads();
  if (w == 0) {
    constexpr uint32_t per = NB / 32;
    uint32_t sum = 0;
    for (uint32_t j = 0; j < per; ++j) sum += cnt[lane * per + j];
    uint32_t inc = sum;
    for (uint32_t o = 1; o < 32; o <<= 1) {
      const uint32_t x = __shfl_up_sync(0xFFFFFFFFu, inc, o);
      if (lane >= o) inc += x;
    }
    uint32_t run = inc - sum;
    for (uint32_t j = 0; j < per; ++j) {
      const uint32_t c = cnt[lane * per + j];
      cnt[lane * per + j] = run;
      run += c;
    }
  }
  __syncthreads();
  for (uint32_t q = t; q < n; q += kOrderThreads) order[atomicAdd(&cnt[cell(q)], 1u)] = q;
}

static const uint32_t* order_by_cell(const DevIndex& ix, const SearchArgs& a, SearchWs& ws, cudaStream_t st) {
  const uint32_t n = a.nwork;
  const size_t o_order = 0, o_proj = ((size_t)n * 4 + 255) / 256 * 256;
  const size_t o_sums = o_proj + ((size_t)n * kSimBits * 4 + 255) / 256 * 256;
  ws.order.ensure(o_sums + 64, st);
  uint8_t* p = (uint8_t*)ws.order.p;
  float* sums = (float*)(p + o_sums);
  GRAB_CUDA(cudaMemsetAsync(sums, 0, kSimBits * 4, st));
  const unsigned blocks = (unsigned)std::min<uint64_t>(div_up(n, 8), 4ull * ix.num_sms);
  k_sim_project<<<blocks, 256, 0, st>>>(a.Q, a.qphys, a.X, a.dp, n, (float*)(p + o_proj), sums);
  GRAB_CHECK_LAUNCH();
  k_order_by_cell<<<1, kOrderThreads, 0, st>>>((const float*)(p + o_proj), sums, n, (uint32_t*)(p + o_order));
  GRAB_CHECK_LAUNCH();
  return (const uint32_t*)(p + o_order);
}

static const uint32_t* order_by_lower(const SearchArgs& a, SearchWs& ws, cudaStream_t st) {
  ws.order.ensure((size_t)a.nwork * 8, st);
  uint32_t* order = (uint32_t*)ws.order.p;
  k_order_by_lower<<<1, kOrderThreads, 0, st>>>(a.lower, a.range_stride, a.nwork, (float*)(order + a.nwork), order);
  GRAB_CHECK_LAUNCH();
  return order;
}

void run_search(const DevIndex& ix, SearchArgs a, cudaStream_t st) {
  if (a.nwork == 0) return;
  reserve_persisting_l2();
  if (a.width * a.k_max > 256) throw Error(GRAB_ERR_VALUE, "search_width * k_max > 256 not supported");
  if (ix.phys_cap >= kExpanded) throw Error(GRAB_ERR_CAPACITY, "search needs phys ids < 2^31");
  ensure_adja(ix, st);
  a.adja = ix.adja;
  SearchShape sh = make_shape(a.itopk, a.width, a.k_max, a.want, a.max_iter, false, a.dp, a.n_live,
                              a.out_stats != nullptr, ix.phys_cap);
  SearchWs& ws = workspace(ix, st);
  std::lock_guard<std::mutex> ws_lock(ws.mu);
  DBufLite& tables = ws.tables;
  DBufLite& big_tables = ws.big_tables;
  DBufLite& ovfb = ws.ovf;
  ovfb.ensure((a.nwork + 1) * sizeof(uint32_t), st);
  uint32_t* ovf = (uint32_t*)ovfb.p;
  GRAB_CUDA(cudaMemsetAsync(ovf, 0, sizeof(uint32_t), st));
  ws.ctr.ensure(2 * sizeof(uint32_t), st);
  uint32_t* ctr = (uint32_t*)ws.ctr.p;
  GRAB_CUDA(cudaMemsetAsync(ctr, 0, 2 * sizeof(uint32_t), st));
  a.work_ctr = getenv("GRAB_STATIC_WORK") ? nullptr : ctr;
  a.ovf_count = ovf;
  a.ovf_list = ovf + 1;
  a.qmap = nullptr;
  a.nwork_dev = nullptr;
  static const bool no_order = getenv("GRAB_SEARCH_NO_ORDER") != nullptr;
  static const bool no_sim = getenv("GRAB_SEARCH_NO_SIM_ORDER") != nullptr;
  if (a.nwork >= kOrderMinQueries && a.work_ctr && !no_order) {
    if (a.range_stride != 0) a.qmap = order_by_lower(a, ws, st);
    else if (!no_sim) a.qmap = order_by_cell(ix, a, ws, st);
  }
#ifdef GRAB_SEARCH_PROFILE
  {
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    GRAB_CUDA(cudaMemcpyToSymbolAsync(g_phase, z, sizeof(z), 0, cudaMemcpyHostToDevice, st));
  }
#endif
  launch(a, sh, ix.num_sms, st, tables, ~0ull);
#ifdef GRAB_SEARCH_PROFILE
  {
    unsigned long long z[8];
    GRAB_CUDA(cudaMemcpyFromSymbolAsync(z, g_phase, sizeof(z), 0, cudaMemcpyDeviceToHost, st));
    GRAB_CUDA(cudaStreamSynchronize(st));
    double tot = 0;
    for (int i = 0; i < 8; ++i) tot += (double)z[i];
    fprintf(stderr, "[grab] search phases %%: setup+seeds %.1f frontier %.1f gather %.1f visited %.1f compact %.1f "
                    "score %.1f admit %.1f output %.1f\n", 100 * z[0] / tot, 100 * z[1] / tot, 100 * z[2] / tot,
            100 * z[3] / tot, 100 * z[4] / tot, 100 * z[5] / tot, 100 * z[6] / tot, 100 * z[7] / tot);
  }
#endif
  SearchShape big = make_shape(a.itopk, a.width, a.k_max, a.want, a.max_iter, true, a.dp, a.n_live,
                               a.out_stats != nullptr, ix.phys_cap);
  // the retry grid's tables: at most ~1 GB (fewer resident warps for huge tables;
  // the grid claims its overflowed queries dynamically, so any size is correct)
  const uint64_t big_warp_bytes = 4ull << big.vlog2;
  const uint64_t big_blocks = std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)ix.num_sms,
                                                                       (1ull << 30) / (4 * big_warp_bytes)));
  SearchArgs b = a;
  b.qmap = a.ovf_list;
  b.nwork_dev = ovf;
  b.ovf_count = nullptr;  // cannot overflow: the table bounds every insert of max_iter iterations
  b.ovf_list = nullptr;
  b.work_ctr = a.work_ctr ? ctr + 1 : nullptr;
  launch(b, big, ix.num_sms, st, big_tables, big_blocks);
  if (getenv("GRAB_DEBUG")) {
    uint32_t n_ovf = 0;
    GRAB_CUDA(cudaMemcpyAsync(&n_ovf, ovf, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    GRAB_CUDA(cudaStreamSynchronize(st));
    fprintf(stderr, "[grab] search nwork=%u vlog2=%u overflow=%u\n", a.nwork, sh.vlog2, n_ovf);
  }
}

}  // namespace grab
