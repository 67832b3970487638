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

// Open-addressing set of 2^lg u32 entries (value key+1, 0 = empty).
// Probe loops are written with a single structured exit: early returns from
// inside a data-dependent loop make the warp look unconverged to the compiler
// and turn every later shuffle into the slow collective fallback.
__device__ __forceinline__ bool set_insert(uint32_t* tab, uint32_t lg, uint32_t key) {
  const uint32_t mask = (1u << lg) - 1;
  uint32_t h = hash32(key) >> (32 - lg);
  const uint32_t v = key + 1;
  uint32_t cur = atomicCAS(tab + h, 0u, v);
  while (cur != 0u && cur != v) {
    h = (h + 1) & mask;
    cur = atomicCAS(tab + h, 0u, v);
  }
  return cur == 0u;
}

__device__ __forceinline__ bool set_contains(const uint32_t* tab, uint32_t lg, uint32_t key) {
  const uint32_t mask = (1u << lg) - 1;
  uint32_t h = hash32(key) >> (32 - lg);
  const uint32_t v = key + 1;
  uint32_t cur = *((volatile const uint32_t*)(tab + h));
  while (cur != 0u && cur != v) {
    h = (h + 1) & mask;
    cur = *((volatile const uint32_t*)(tab + h));
  }
  return cur == v;
}

__device__ __forceinline__ void clear_words(uint32_t* p, uint32_t n) {
  // n is a multiple of 128 (4 words per lane per step)
  const uint4 z = make_uint4(0, 0, 0, 0);
  for (uint32_t i = lane_id() * 4; i < n; i += 128) *reinterpret_cast<uint4*>(p + i) = z;
}

// ---------------------------------------------------------------- layout
__host__ __device__ inline uint32_t align16(uint32_t x) { return (x + 15u) & ~15u; }

struct WarpLayout {
  uint32_t qd, qs, qp, qf, cd, cs, cp, dd, fr, bytes;
};

__host__ __device__ inline WarpLayout warp_layout(const SearchShape& s) {
  WarpLayout l;
  uint32_t o = 0;
  l.qd = o;
  o += align16(s.itopk * 8);
  l.cd = o;
  o += align16(s.cmax * 8);
  l.qs = o;
  o += align16(s.itopk * 4);
  l.qp = o;
  o += align16(s.itopk * 4);
  l.cs = o;
  o += align16(s.cmax * 4);
  l.cp = o;
  o += align16(s.cmax * 4);
  l.dd = o;
  o += align16(s.dsz * 4);
  l.fr = o;
  o += align16(s.width * 4);
  l.qf = o;
  o += align16(s.itopk);
  l.bytes = o;
  return l;
}

// ---------------------------------------------------------------- distances
template <int NC>
struct QueryRegs {
  float4 q[NC];
};

template <int NC>
__device__ __forceinline__ void load_query(QueryRegs<NC>& r, const float* q, uint32_t dp) {
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const uint32_t col = (c * 32 + lane_id()) * 4;
    r.q[c] = col < dp ? *reinterpret_cast<const float4*>(q + col) : make_float4(0, 0, 0, 0);
  }
}

template <int NC>
struct GroupOf {
  static constexpr int G = NC == 1 ? 8 : (NC == 2 ? 4 : (NC <= 4 ? 2 : 1));
};

// Distances for cand[0..n): writes cd[i]. All lanes participate.
template <int NC>
__device__ __forceinline__ void score(const QueryRegs<NC>& qr, const float* __restrict__ X, uint32_t dp,
                                      const uint32_t* cp, double* cd, uint32_t n) {
  constexpr int G = GroupOf<NC>::G;
  const uint32_t lane = lane_id();
  for (uint32_t base = 0; base < n; base += G) {
    float4 x[G][NC];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const uint32_t i = base + g;
      const uint32_t p = cp[i < n ? i : base];
      const float* row = X + (uint64_t)p * dp;
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const uint32_t col = (c * 32 + lane) * 4;
        x[g][c] = col < dp ? ldg_nc_f4(row + col) : make_float4(0, 0, 0, 0);
      }
    }
    double part[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      double acc = 0.0;
#pragma unroll
      for (int c = 0; c < NC; ++c) acc = sq4(x[g][c], qr.q[c], acc);
      part[g] = acc;
    }
    const double v = reduce_scatter<G>(part);
    constexpr uint32_t SPAN = 32 / G;  // lanes holding each candidate's sum
    const uint32_t g = lane / SPAN;
    if ((lane % SPAN) == 0 && base + g < n) cd[base + g] = v;
  }
  __syncwarp();
}

// ---------------------------------------------------------------- queue ops
__device__ __forceinline__ void bitonic_sort(double* d, uint32_t* s, uint32_t* p, uint32_t n, uint32_t P) {
  const uint32_t lane = lane_id();
  for (uint32_t i = n + lane; i < P; i += 32) {
    d[i] = __longlong_as_double(0x7FF0000000000000ll);  // +inf
    s[i] = 0xFFFFFFFFu;
    p[i] = 0xFFFFFFFFu;
  }
  __syncwarp();
  for (uint32_t k = 2; k <= P; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t i = lane; i < P; i += 32) {
        const uint32_t l = i ^ j;
        if (l > i) {
          const double di = d[i], dl = d[l];
          const uint32_t si = s[i], sl = s[l];
          const bool asc = (i & k) == 0;
          if (key_less(dl, sl, di, si) == asc) {
            d[i] = dl;
            d[l] = di;
            s[i] = sl;
            s[l] = si;
            const uint32_t t = p[i];
            p[i] = p[l];
            p[l] = t;
          }
        }
      }
      __syncwarp();
    }
  }
}

// number of entries in sorted (d,s)[0..n) strictly less than key
__device__ __forceinline__ uint32_t rank_in(const double* d, const uint32_t* s, uint32_t n, double kd, uint32_t ks) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (key_less(d[mid], s[mid], kd, ks))
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

// CandidateQueue.admit: merge cand[0..nc) into the queue (length L) in place,
// truncated to itopk. Returns the new length.
__device__ __forceinline__ uint32_t admit(double* qd, uint32_t* qs, uint32_t* qp, uint8_t* qf, double* cd,
                                          uint32_t* cs, uint32_t* cp, uint32_t L, uint32_t nc, uint32_t itopk) {
  const uint32_t lane = lane_id();
  if (L == itopk && nc) {  // candidates that cannot survive truncation are dropped up front
    const double td = qd[L - 1];
    const uint32_t ts = qs[L - 1];
    uint32_t kept = 0;
    for (uint32_t b0 = 0; b0 < nc; b0 += 32) {
      const uint32_t i = b0 + lane;
      bool ok = false;
      double d = 0;
      uint32_t s = 0, p = 0;
      if (i < nc) {
        d = cd[i];
        s = cs[i];
        p = cp[i];
        ok = key_less(d, s, td, ts);
      }
      const uint32_t m = __ballot_sync(0xFFFFFFFFu, ok);
      __syncwarp();
      if (ok) {
        const uint32_t pos = kept + __popc(m & ((1u << lane) - 1));
        cd[pos] = d;
        cs[pos] = s;
        cp[pos] = p;
      }
      kept += __popc(m);
      __syncwarp();
    }
    nc = kept;
  }
  if (nc == 0) return L;
  uint32_t P = 32;
  while (P < nc) P <<= 1;
  bitonic_sort(cd, cs, cp, nc, P);
  // candidate destinations against the OLD queue (<= 4 per lane, cmax <= 128 on this path)
  uint32_t cpos[4];
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const uint32_t j = lane + 32 * t;
    cpos[t] = j < nc ? j + rank_in(qd, qs, L, cd[j], cs[j]) : 0xFFFFFFFFu;
  }
  // move queue entries, highest chunk first (destinations are >= sources)
  for (int32_t b0 = (int32_t)((L - 1) & ~31u); b0 >= 0; b0 -= 32) {
    const uint32_t i = (uint32_t)b0 + lane;
    double d = 0;
    uint32_t s = 0, p = 0, pos = 0xFFFFFFFFu;
    uint8_t f = 0;
    if (i < L) {
      d = qd[i];
      s = qs[i];
      p = qp[i];
      f = qf[i];
      pos = i + rank_in(cd, cs, nc, d, s);
    }
    __syncwarp();
    if (pos < itopk) {
      qd[pos] = d;
      qs[pos] = s;
      qp[pos] = p;
      qf[pos] = f;
    }
    __syncwarp();
  }
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const uint32_t j = lane + 32 * t;
    if (cpos[t] < itopk) {
      qd[cpos[t]] = cd[j];
      qs[cpos[t]] = cs[j];
      qp[cpos[t]] = cp[j];
      qf[cpos[t]] = 0;
    }
  }
  __syncwarp();
  return min(itopk, L + nc);
}

// ---------------------------------------------------------------- seeds
// _sample_seeds (searcher.py:101-153). Draws of one jump-ahead round (64 words,
// lane L owns output 32r+L = words lo,hi) are compacted into `stage` in word
// order, then consumed 32 at a time in draw order. Returns seeds written to
// (cp, cs)[0..n); *attempts = SearchStats.seed_attempts.
__device__ uint32_t sample_seeds(const SearchArgs& a, uint32_t* stage, uint32_t* cp, uint32_t* cs, uint32_t* vis,
                                 uint32_t vlg, uint32_t lo_b, uint32_t hi_b, float lo_f, float hi_f,
                                 uint64_t rng_seed, uint32_t* attempts) {
  const uint32_t lane = lane_id();
  const uint32_t lt = (1u << lane) - 1;
  const uint32_t want = a.want;
  const uint64_t c0 = a.bcum[lo_b];
  const uint64_t total = a.bcum[hi_b + 1] - c0;
  uint32_t picked = 0;
  *attempts = 0;
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
          uint32_t lo = lo_b, hi = hi_b;  // bucket b with bcum[b] <= f < bcum[b+1]
          while (lo < hi) {
            const uint32_t mid = (lo + hi + 1) >> 1;
            if (__ldg(a.bcum + mid) <= f)
              lo = mid;
            else
              hi = mid - 1;
          }
          phys = __ldg(a.bstart + lo) + (uint32_t)(f - __ldg(a.bcum + lo));
          const Attr at = ld_attr(a.attr, phys);
          slot = at.slot;
          sv = at.s;
        }
        const bool inr = have && slot < a.n_live && sv >= lo_f && sv <= hi_f;
        const uint32_t same = __match_any_sync(0xFFFFFFFFu, inr ? phys : 0xFFFFFFFFu);
        const bool first = inr && (uint32_t)(__ffs(same) - 1) == lane;
        const bool fresh = first && !set_contains(vis, vlg, phys);
        const uint32_t fm = __ballot_sync(0xFFFFFFFFu, fresh);
        const uint32_t rank = __popc(fm & lt);
        const bool take = fresh && rank < want - picked;
        if (take) {
          set_insert(vis, vlg, phys);
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
          ok = slot < a.n_live && at.s >= lo_f && at.s <= hi_f && !set_contains(vis, vlg, phys);
        }
        const uint32_t msk = __ballot_sync(0xFFFFFFFFu, ok);
        const uint32_t rank = __popc(msk & lt);
        const bool take = ok && rank < want - picked;
        if (take) {
          set_insert(vis, vlg, phys);
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

// ---------------------------------------------------------------- kernel
// NC: 128-float chunks per row; EPL: gathered neighbours per lane per iteration
// (width * K_max <= 32 * EPL).
#ifndef GRAB_SEARCH_MINB
#define GRAB_SEARCH_MINB 6  // 6 blocks x 4 warps: 85 registers (small spills beat 4 blocks)
#endif
template <int NC, int EPL>
__global__ void __launch_bounds__(128, GRAB_SEARCH_MINB) k_search(SearchArgs a, SearchShape sh) {
  extern __shared__ __align__(16) uint8_t smem[];
  const uint32_t lane = lane_id();
  const uint32_t wib = threadIdx.x >> 5;
  const uint32_t wpb = blockDim.x >> 5;
  const WarpLayout lay = warp_layout(sh);
  uint8_t* base = smem + wib * lay.bytes;
  double* qd = (double*)(base + lay.qd);
  uint32_t* qs = (uint32_t*)(base + lay.qs);
  uint32_t* qp = (uint32_t*)(base + lay.qp);
  uint8_t* qf = base + lay.qf;
  double* cd = (double*)(base + lay.cd);
  uint32_t* cs = (uint32_t*)(base + lay.cs);
  uint32_t* cp = (uint32_t*)(base + lay.cp);
  uint32_t* dd = (uint32_t*)(base + lay.dd);
  uint32_t* fr = (uint32_t*)(base + lay.fr);
  const uint32_t gw = blockIdx.x * wpb + wib;
  const uint32_t vlg = sh.vlog2;
  uint32_t* vis = a.gtab + ((uint64_t)gw << vlg);
  const uint32_t vcap = (1u << vlg) / 4 * 3;
  const uint32_t nw = gridDim.x * wpb;
  const uint32_t dlg = 31 - __clz(sh.dsz);
  const uint32_t K = a.k_max;

  for (uint32_t item = gw; item < a.nwork; item += nw) {
    const uint32_t qi = a.qmap ? a.qmap[item] : item;
    const float lo_f = __double2float_rn(a.lower[(uint64_t)qi * a.range_stride]);
    const float hi_f = __double2float_rn(a.upper[(uint64_t)qi * a.range_stride]);
    grab_search_stats st = {0, 0, 0, 0, 0, 0, 0, 0};
    uint32_t L = 0;
    bool overflow = false;
    if (a.n_live > 0 && a.m > 0) {
      clear_words(vis, 1u << vlg);
      __syncwarp();
      QueryRegs<NC> qr;
      load_query<NC>(qr, a.qphys ? a.X + (uint64_t)a.qphys[qi] * a.dp : a.Q + (uint64_t)qi * a.dp, a.dp);
      const uint32_t lo_b = bucket_of_f32(a.bound, a.m, lo_f);
      const uint32_t hi_b = bucket_of_f32(a.bound, a.m, hi_f);
      const uint64_t seed = a.seeds ? a.seeds[qi] : derive_query_seed(a.seed_base, a.ordinal0 + qi);
      uint32_t attempts = 0;
      const uint32_t ns = sample_seeds(a, dd, cp, cs, vis, vlg, lo_b, hi_b, lo_f, hi_f, seed, &attempts);
      st.seed_attempts = attempts;
      uint32_t vis_n = ns;
      if (ns > 0) {
        score<NC>(qr, a.X, a.dp, cp, cd, ns);
        st.dist_evals = st.seed_evals = ns;
        L = admit(qd, qs, qp, qf, cd, cs, cp, 0, ns, sh.itopk);
        for (uint32_t it = 0; it < a.max_iter; ++it) {
          // frontier: first `width` unexpanded entries
          uint32_t nf = 0;
          for (uint32_t b0 = 0; b0 < L && nf < sh.width; b0 += 32) {
            const uint32_t i = b0 + lane;
            const bool un = i < L && qf[i] == 0;
            const uint32_t m = __ballot_sync(0xFFFFFFFFu, un);
            const uint32_t rank = __popc(m & ((1u << lane) - 1));
            if (un && nf + rank < sh.width) {
              fr[nf + rank] = qp[i];
              qf[i] = 1;
            }
            nf = min(sh.width, nf + __popc(m));
          }
          __syncwarp();
          if (nf == 0) break;
          const uint32_t fan = nf * K;
          if (vis_n + fan > vcap) {
            overflow = true;
            break;
          }
          st.iterations++;
          st.expanded += nf;
          clear_words(dd, sh.dsz);
          // (1) all adjacency entries of the frontier rows
          uint32_t v[EPL];
#pragma unroll
          for (int t = 0; t < EPL; ++t) {
            const uint32_t e = lane + 32 * t;
            v[t] = kSentinel;
            if (e < fan) v[t] = __ldg(a.adj + (uint64_t)fr[e / K] * K + (e % K));
          }
          // (2) all Attr{scalar, slot}
          float sv[EPL];
          uint32_t sl[EPL];
#pragma unroll
          for (int t = 0; t < EPL; ++t) {
            sl[t] = kNoSlot;
            sv[t] = 0.f;
            if (v[t] != kSentinel) {
              const Attr at = ld_attr(a.attr, v[t]);
              sl[t] = at.slot;
              sv[t] = at.s;
            }
          }
          __syncwarp();
          // (3) per-iteration unique (shared), pre-check, (4) visited CAS (global)
          uint32_t uniq_bits = 0, cand_bits = 0, rej_bits = 0;
#pragma unroll
          for (int t = 0; t < EPL; ++t) {
            if (sl[t] < a.n_live && set_insert(dd, dlg, v[t])) {
              uniq_bits |= 1u << t;
              if (sv[t] >= lo_f && sv[t] <= hi_f)
                cand_bits |= 1u << t;
              else
                rej_bits |= 1u << t;
            }
          }
          {
            // issue every first-probe CAS of the iteration before consuming any
            const uint32_t vmask = (1u << vlg) - 1;
            uint32_t h[EPL], cur[EPL];
#pragma unroll
            for (int t = 0; t < EPL; ++t) {
              h[t] = hash32(v[t]) >> (32 - vlg);
              cur[t] = ((cand_bits >> t) & 1u) ? atomicCAS(vis + h[t], 0u, v[t] + 1) : 0u;
            }
#pragma unroll
            for (int t = 0; t < EPL; ++t) {
              if ((cand_bits >> t) & 1u) {
                while (cur[t] != 0u && cur[t] != v[t] + 1) {  // rare collision: probe on
                  h[t] = (h[t] + 1) & vmask;
                  cur[t] = atomicCAS(vis + h[t], 0u, v[t] + 1);
                }
                if (cur[t] != 0u) cand_bits &= ~(1u << t);
              }
            }
          }
          // (5) compact candidates in gather order + stats
          uint32_t nc = 0;
#pragma unroll
          for (int t = 0; t < EPL; ++t) {
            const bool c = (cand_bits >> t) & 1u;
            const uint32_t cm = __ballot_sync(0xFFFFFFFFu, c);
            st.gathered += __popc(__ballot_sync(0xFFFFFFFFu, (uniq_bits >> t) & 1u));
            st.precheck_rejected += __popc(__ballot_sync(0xFFFFFFFFu, (rej_bits >> t) & 1u));
            if (c) {
              const uint32_t pos = nc + __popc(cm & ((1u << lane) - 1));
              cp[pos] = v[t];
              cs[pos] = sl[t];
            }
            nc += __popc(cm);
          }
          __syncwarp();
          vis_n += nc;
          if (nc == 0) continue;
          st.in_range_new += nc;
          st.dist_evals += nc;
          score<NC>(qr, a.X, a.dp, cp, cd, nc);
          L = admit(qd, qs, qp, qf, cd, cs, cp, L, nc, sh.itopk);
        }
      }
    }
    if (overflow) {
      if (lane == 0) {
        const uint32_t pos = atomicAdd(a.ovf_count, 1u);
        a.ovf_list[pos] = qi;
      }
      __syncwarp();
      continue;
    }
    const uint32_t cnt = min(L, a.k);
    for (uint32_t i = lane; i < a.k; i += 32) {
      a.out_slots[(uint64_t)qi * a.k + i] = i < cnt ? (int64_t)qs[i] : -1;
      a.out_dists[(uint64_t)qi * a.k + i] = i < cnt ? qd[i] : __longlong_as_double(0x7FF8000000000000ll);
    }
    if (lane == 0) {
      a.out_counts[qi] = cnt;
      if (a.out_stats) a.out_stats[qi] = st;
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------- host
static uint32_t ceil_log2(uint64_t x) {
  uint32_t l = 0;
  while ((1ull << l) < x) ++l;
  return l;
}

SearchShape make_shape(uint32_t itopk, uint32_t width, uint32_t k_max, uint32_t want, uint32_t max_iter, bool worst) {
  SearchShape s;
  s.itopk = itopk;
  s.width = width;
  const uint32_t fan = width * k_max;
  s.cmax = 1u << ceil_log2(std::max<uint64_t>(std::max(fan, want), 32));  // bitonic pads to a power of 2
  s.dsz = 1u << ceil_log2(std::max<uint64_t>(2ull * fan, 128));
  if (!worst) {
    s.vlog2 = std::min<uint32_t>(15, std::max<uint32_t>(11, ceil_log2((uint64_t)itopk * 24)));
  } else {
    const uint64_t bound = (uint64_t)want + (uint64_t)max_iter * fan + fan;
    s.vlog2 = std::max<uint32_t>(11, ceil_log2(bound * 4 / 3 + 1));
  }
  return s;
}

// returns the number of warps the grid runs (for sizing the visited tables)
template <int NC, int EPL>
static void launch_t(const SearchArgs& a, const SearchShape& sh, uint32_t wpb, uint32_t blocks, uint32_t smem,
                     cudaStream_t st) {
  auto kern = k_search<NC, EPL>;
  GRAB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern<<<blocks, 32 * wpb, smem, st>>>(a, sh);
  GRAB_CHECK_LAUNCH();
}

template <int NC>
static void dispatch_epl(uint32_t epl, const SearchArgs& a, const SearchShape& sh, uint32_t wpb, uint32_t blocks,
                         uint32_t smem, cudaStream_t st) {
  if (epl <= 1)
    launch_t<NC, 1>(a, sh, wpb, blocks, smem, st);
  else if (epl <= 2)
    launch_t<NC, 2>(a, sh, wpb, blocks, smem, st);
  else if (epl <= 4)
    launch_t<NC, 4>(a, sh, wpb, blocks, smem, st);
  else
    throw Error(GRAB_ERR_VALUE, "search_width * k_max > 128 not supported");
}

static int occupancy_blocks(uint32_t nc, uint32_t epl, uint32_t wpb, uint32_t smem) {
  int per_sm = 0;
  auto q = [&](auto kern) {
    GRAB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    GRAB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * wpb, smem));
  };
  // occupancy depends on registers (template) and smem; probe the instance that will run
#define GRAB_Q(NC_, EPL_) \
  if (nc == NC_ && epl == EPL_) q(k_search<NC_, EPL_>);
  GRAB_Q(1, 1) GRAB_Q(1, 2) GRAB_Q(1, 4) GRAB_Q(2, 1) GRAB_Q(2, 2) GRAB_Q(2, 4) GRAB_Q(4, 1) GRAB_Q(4, 2)
  GRAB_Q(4, 4) GRAB_Q(8, 1) GRAB_Q(8, 2) GRAB_Q(8, 4)
#undef GRAB_Q
  return per_sm < 1 ? 1 : per_sm;
}

static void launch(SearchArgs a, const SearchShape& sh, int num_sms, cudaStream_t st, DBufLite& tables) {
  const WarpLayout lay = warp_layout(sh);
  const uint32_t wpb = 4;
  const uint32_t smem = lay.bytes * wpb;
  if (smem > 227 * 1024) throw Error(GRAB_ERR_VALUE, "search parameters exceed shared memory (itopk too large)");
  uint32_t nc = (uint32_t)div_up(a.dp, 128);
  nc = nc <= 1 ? 1 : nc <= 2 ? 2 : nc <= 4 ? 4 : nc <= 8 ? 8 : 0;
  if (!nc) throw Error(GRAB_ERR_VALUE, "dimension > 1024 not supported by the search kernel");
  uint32_t epl = (uint32_t)div_up(sh.width * a.k_max, 32);
  epl = epl <= 1 ? 1 : epl <= 2 ? 2 : epl <= 4 ? 4 : 8;
  if (epl > 4 || sh.cmax > 128) throw Error(GRAB_ERR_VALUE, "search_width * k_max > 128 not supported");
  const int per_sm = occupancy_blocks(nc, epl, wpb, smem);
  const uint64_t blocks = std::min<uint64_t>(div_up(a.nwork, wpb), (uint64_t)per_sm * num_sms);
  if (!blocks) return;
  // one visited table per resident warp
  const uint64_t words = blocks * wpb * (1ull << sh.vlog2);
  tables.ensure(words * 4, st);
  a.gtab = (uint32_t*)tables.p;
  if (nc == 1)
    dispatch_epl<1>(epl, a, sh, wpb, (uint32_t)blocks, smem, st);
  else if (nc == 2)
    dispatch_epl<2>(epl, a, sh, wpb, (uint32_t)blocks, smem, st);
  else if (nc == 4)
    dispatch_epl<4>(epl, a, sh, wpb, (uint32_t)blocks, smem, st);
  else
    dispatch_epl<8>(epl, a, sh, wpb, (uint32_t)blocks, smem, st);
}

void run_search(const DevIndex& ix, SearchArgs a, cudaStream_t st) {
  if (a.nwork == 0) return;
  if (a.width * a.k_max > 128) throw Error(GRAB_ERR_VALUE, "search_width * k_max > 128 not supported");
  SearchShape sh = make_shape(a.itopk, a.width, a.k_max, a.want, a.max_iter, false);
  DBufLite tables, ovfb;
  ovfb.ensure((a.nwork + 1) * sizeof(uint32_t), st);
  uint32_t* ovf = (uint32_t*)ovfb.p;
  GRAB_CUDA(cudaMemsetAsync(ovf, 0, sizeof(uint32_t), st));
  a.ovf_count = ovf;
  a.ovf_list = ovf + 1;
  a.qmap = nullptr;
  launch(a, sh, ix.num_sms, st, tables);
  uint32_t n_ovf = 0;
  GRAB_CUDA(cudaMemcpyAsync(&n_ovf, ovf, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
  GRAB_CUDA(cudaStreamSynchronize(st));
  if (getenv("GRAB_DEBUG")) fprintf(stderr, "[grab] search nwork=%u vlog2=%u overflow=%u\n", a.nwork, sh.vlog2, n_ovf);
  if (n_ovf) {
    // exact re-run of the overflowed queries with a worst-case visited table
    SearchShape big = make_shape(a.itopk, a.width, a.k_max, a.want, a.max_iter, true);
    SearchArgs b = a;
    DBufLite qm;
    qm.ensure(n_ovf * sizeof(uint32_t), st);
    GRAB_CUDA(cudaMemcpyAsync(qm.p, a.ovf_list, n_ovf * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st));
    b.qmap = (const uint32_t*)qm.p;
    b.nwork = n_ovf;
    GRAB_CUDA(cudaMemsetAsync(ovf, 0, sizeof(uint32_t), st));
    launch(b, big, ix.num_sms, st, tables);
    uint32_t again = 0;
    GRAB_CUDA(cudaMemcpyAsync(&again, ovf, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    GRAB_CUDA(cudaStreamSynchronize(st));
    if (again) throw Error(GRAB_ERR_CUDA, "visited-set overflow persisted on the worst-case retry");
  }
}

}  // namespace grab
