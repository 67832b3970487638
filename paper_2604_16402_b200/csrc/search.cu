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
// B200 mapping: a persistent grid of warps, each owning one query at a time.
// Query vector lives in registers (float4 per lane per 128-float chunk);
// candidate rows are fetched with 16-byte ld.global.nc, G rows in flight per
// lane, reduced with one fixed xor tree in f64 (parity with the reference's
// f64 accumulation). Queue, candidate buffer, per-iteration dedup table and
// the exact visited hash set live in shared memory; the visited set is
// speculatively sized and a query that would exceed 3/4 load is re-run with
// a table sized for the worst case (never a forgetful hash).
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

// insert phys id into an open-addressing set of 2^lg entries (0 = empty).
// Returns true when newly inserted.
__device__ __forceinline__ bool set_insert(uint32_t* tab, uint32_t lg, uint32_t key) {
  uint32_t mask = (1u << lg) - 1;
  uint32_t h = hash32(key) >> (32 - lg);
  uint32_t v = key + 1;
  while (true) {
    uint32_t cur = atomicCAS(tab + h, 0u, v);
    if (cur == 0u) return true;
    if (cur == v) return false;
    h = (h + 1) & mask;
  }
}

__device__ __forceinline__ bool set_contains(const uint32_t* tab, uint32_t lg, uint32_t key) {
  uint32_t mask = (1u << lg) - 1;
  uint32_t h = hash32(key) >> (32 - lg);
  uint32_t v = key + 1;
  while (true) {
    uint32_t cur = *((volatile const uint32_t*)(tab + h));
    if (cur == v) return true;
    if (cur == 0u) return false;
    h = (h + 1) & mask;
  }
}

__device__ __forceinline__ void clear_words(uint32_t* p, uint32_t n) {
  // n is a multiple of 128 (4 words per lane per step)
  uint4 z = make_uint4(0, 0, 0, 0);
  for (uint32_t i = lane_id() * 4; i < n; i += 128) *reinterpret_cast<uint4*>(p + i) = z;
}

struct WarpSmem {
  double* qd[2];
  uint32_t* qs[2];
  uint32_t* qp[2];
  uint8_t* qf[2];
  double* cd;
  uint32_t* cs;
  uint32_t* cp;
  uint32_t* dedup;
  uint32_t* fr;
  uint32_t* vis;
};

__host__ __device__ inline uint32_t align8(uint32_t x) { return (x + 7u) & ~7u; }

__host__ __device__ inline uint32_t warp_smem_bytes(const SearchShape& s, bool vis_in_smem) {
  uint32_t b = 0;
  b += 2 * align8(s.itopk * 8);
  b += 2 * align8(s.itopk * 4) * 2;
  b += 2 * align8(s.itopk);
  b += align8(s.cmax * 8) + 2 * align8(s.cmax * 4);
  b += align8(s.dsz * 4);
  b += align8(s.width * 4);
  b = (b + 15u) & ~15u;
  if (vis_in_smem) b += (1u << s.vlog2) * 4;
  return b;
}

__device__ inline WarpSmem carve(uint8_t* base, const SearchShape& s) {
  WarpSmem w;
  uint8_t* p = base;
  for (int i = 0; i < 2; ++i) {
    w.qd[i] = (double*)p;
    p += align8(s.itopk * 8);
  }
  for (int i = 0; i < 2; ++i) {
    w.qs[i] = (uint32_t*)p;
    p += align8(s.itopk * 4);
    w.qp[i] = (uint32_t*)p;
    p += align8(s.itopk * 4);
  }
  for (int i = 0; i < 2; ++i) {
    w.qf[i] = p;
    p += align8(s.itopk);
  }
  w.cd = (double*)p;
  p += align8(s.cmax * 8);
  w.cs = (uint32_t*)p;
  p += align8(s.cmax * 4);
  w.cp = (uint32_t*)p;
  p += align8(s.cmax * 4);
  w.dedup = (uint32_t*)p;
  p += align8(s.dsz * 4);
  w.fr = (uint32_t*)p;
  p += align8(s.width * 4);
  p = (uint8_t*)(((uintptr_t)p + 15) & ~(uintptr_t)15);
  w.vis = (uint32_t*)p;
  return w;
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
    uint32_t col = (c * 32 + lane_id()) * 4;
    r.q[c] = col < dp ? *reinterpret_cast<const float4*>(q + col) : make_float4(0, 0, 0, 0);
  }
}

template <int NC>
struct GroupOf {
  static constexpr int G = NC == 1 ? 8 : (NC == 2 ? 4 : (NC <= 4 ? 2 : 1));
};

// Distances for cand[0..n): writes cd[i]. All lanes participate.
template <int NC>
__device__ __forceinline__ void score(const QueryRegs<NC>& qr, const float* X, uint32_t dp, const uint32_t* cp,
                                      double* cd, uint32_t n) {
  constexpr int G = GroupOf<NC>::G;
  const uint32_t lane = lane_id();
  for (uint32_t base = 0; base < n; base += G) {
    float4 x[G][NC];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      uint32_t i = base + g;
      uint32_t p = i < n ? cp[i] : cp[0];
      const float* row = X + (uint64_t)p * dp;
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        uint32_t col = (c * 32 + lane) * 4;
        x[g][c] = col < dp ? ldg_nc_f4(row + col) : make_float4(0, 0, 0, 0);
      }
    }
#pragma unroll
    for (int g = 0; g < G; ++g) {
      double acc = 0.0;
#pragma unroll
      for (int c = 0; c < NC; ++c) acc = sq4(x[g][c], qr.q[c], acc);
      acc = warp_sum(acc);
      if (lane == 0 && base + g < n) cd[base + g] = acc;
    }
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
        uint32_t l = i ^ j;
        if (l > i) {
          double di = d[i], dl = d[l];
          uint32_t si = s[i], sl = s[l];
          bool asc = (i & k) == 0;
          bool gt = key_less(dl, sl, di, si);  // element i > element l
          if (gt == asc) {
            d[i] = dl;
            d[l] = di;
            s[i] = sl;
            s[l] = si;
            uint32_t t = p[i];
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
    uint32_t mid = (lo + hi) >> 1;
    if (key_less(d[mid], s[mid], kd, ks))
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

// Admit cand[0..nc) into queue buffer `cur` of length L (CandidateQueue.admit).
// Returns new length; flips `cur`.
__device__ uint32_t admit(WarpSmem& w, int& cur, uint32_t L, uint32_t nc, uint32_t itopk) {
  const uint32_t lane = lane_id();
  double* qd = w.qd[cur];
  uint32_t* qs = w.qs[cur];
  // candidates that cannot survive truncation are dropped up front
  if (L == itopk && nc) {
    double td = qd[L - 1];
    uint32_t ts = qs[L - 1];
    uint32_t kept = 0;
    for (uint32_t b0 = 0; b0 < nc; b0 += 32) {
      uint32_t i = b0 + lane;
      bool ok = false;
      double d = 0;
      uint32_t s = 0, p = 0;
      if (i < nc) {
        d = w.cd[i];
        s = w.cs[i];
        p = w.cp[i];
        ok = key_less(d, s, td, ts);
      }
      uint32_t m = __ballot_sync(0xFFFFFFFFu, ok);
      __syncwarp();
      if (ok) {
        uint32_t pos = kept + __popc(m & ((1u << lane) - 1));
        w.cd[pos] = d;
        w.cs[pos] = s;
        w.cp[pos] = p;
      }
      kept += __popc(m);
      __syncwarp();
    }
    nc = kept;
  }
  if (nc == 0) return L;
  uint32_t P = 32;
  while (P < nc) P <<= 1;
  bitonic_sort(w.cd, w.cs, w.cp, nc, P);
  int nxt = cur ^ 1;
  double* od = w.qd[nxt];
  uint32_t* os = w.qs[nxt];
  uint32_t* op = w.qp[nxt];
  uint8_t* of = w.qf[nxt];
  for (uint32_t i = lane; i < L; i += 32) {
    uint32_t pos = i + rank_in(w.cd, w.cs, nc, qd[i], qs[i]);
    if (pos < itopk) {
      od[pos] = qd[i];
      os[pos] = qs[i];
      op[pos] = w.qp[cur][i];
      of[pos] = w.qf[cur][i];
    }
  }
  for (uint32_t j = lane; j < nc; j += 32) {
    uint32_t pos = j + rank_in(qd, qs, L, w.cd[j], w.cs[j]);
    if (pos < itopk) {
      od[pos] = w.cd[j];
      os[pos] = w.cs[j];
      op[pos] = w.cp[j];
      of[pos] = 0;
    }
  }
  __syncwarp();
  cur = nxt;
  return min(itopk, L + nc);
}

// ---------------------------------------------------------------- seeds
struct SeedOut {
  uint32_t n;         // seeds written to cand[0..n)
  uint32_t attempts;  // draws requested (SearchStats.seed_attempts)
};

// _sample_seeds (searcher.py:101-153). Draws of one jump-ahead round (64 words,
// lane L owns output 32r+L = words lo,hi) are compacted into `stage` in word
// order, then consumed 32 at a time in draw order.
__device__ SeedOut sample_seeds(const SearchArgs& a, WarpSmem& w, uint32_t lo_b, uint32_t hi_b, float lo_f,
                                float hi_f, uint64_t rng_seed, uint32_t vlg) {
  const uint32_t lane = lane_id();
  const uint32_t lt = (1u << lane) - 1;
  const uint32_t want = a.want;
  uint32_t* stage = w.dedup;  // >= 128 words, idle during seeding
  SeedOut r{0, 0};
  const uint64_t c0 = a.bcum[lo_b];
  const uint64_t total = a.bcum[hi_b + 1] - c0;
  uint32_t picked = 0;
  if (total > 0) {
    const uint32_t ndraw = 4 * want;
    r.attempts = ndraw;
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
            uint32_t mid = (lo + hi + 1) >> 1;
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
        const bool fresh = first && !set_contains(w.vis, vlg, phys);
        const uint32_t fm = __ballot_sync(0xFFFFFFFFu, fresh);
        const uint32_t rank = __popc(fm & lt);
        const bool take = fresh && rank < want - picked;
        if (take) {
          set_insert(w.vis, vlg, phys);
          w.cp[picked + rank] = phys;
          w.cs[picked + rank] = slot;
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
          ok = slot < a.n_live && at.s >= lo_f && at.s <= hi_f && !set_contains(w.vis, vlg, phys);
        }
        const uint32_t msk = __ballot_sync(0xFFFFFFFFu, ok);
        const uint32_t rank = __popc(msk & lt);
        const bool take = ok && rank < want - picked;
        if (take) {
          set_insert(w.vis, vlg, phys);
          w.cp[picked + rank] = phys;
          w.cs[picked + rank] = slot;
        }
        picked += __popc(__ballot_sync(0xFFFFFFFFu, take));
        __syncwarp();
      }
    }
  }
  r.n = picked;
  return r;
}

// ---------------------------------------------------------------- kernel
template <int NC>
__global__ void __launch_bounds__(128) k_search(SearchArgs a, SearchShape sh) {
  extern __shared__ __align__(16) uint8_t smem[];
  const uint32_t lane = lane_id();
  const uint32_t wib = threadIdx.x >> 5;
  const uint32_t wpb = blockDim.x >> 5;
  const bool vis_smem = a.gtab == nullptr;
  const uint32_t wbytes = warp_smem_bytes(sh, vis_smem);
  WarpSmem w = carve(smem + wib * wbytes, sh);
  const uint32_t gw = blockIdx.x * wpb + wib;
  if (!vis_smem) w.vis = a.gtab + (uint64_t)gw * (1u << sh.vlog2);
  const uint32_t vlg = sh.vlog2;
  const uint32_t vcap = (1u << vlg) / 4 * 3;
  const uint32_t nw = gridDim.x * wpb;

  for (uint32_t item = gw; item < a.nwork; item += nw) {
    const uint32_t qi = a.qmap ? a.qmap[item] : item;
    const double lo_d = a.lower[(uint64_t)qi * a.range_stride];
    const double hi_d = a.upper[(uint64_t)qi * a.range_stride];
    const float lo_f = __double2float_rn(lo_d), hi_f = __double2float_rn(hi_d);
    grab_search_stats st = {0, 0, 0, 0, 0, 0, 0, 0};
    uint32_t L = 0;
    int cur = 0;
    bool overflow = false;
    if (a.n_live > 0 && a.m > 0) {
      clear_words(w.vis, 1u << vlg);
      __syncwarp();
      QueryRegs<NC> qr;
      load_query<NC>(qr, a.qphys ? a.X + (uint64_t)a.qphys[qi] * a.dp : a.Q + (uint64_t)qi * a.dp, a.dp);
      const uint32_t lo_b = bucket_of_f32(a.bound, a.m, lo_f);
      const uint32_t hi_b = bucket_of_f32(a.bound, a.m, hi_f);
      const uint64_t seed = a.seeds ? a.seeds[qi] : derive_query_seed(a.seed_base, a.ordinal0 + qi);
      SeedOut so = sample_seeds(a, w, lo_b, hi_b, lo_f, hi_f, seed, vlg);
      st.seed_attempts = so.attempts;
      uint32_t vis_n = so.n;
      if (so.n > 0) {
        score<NC>(qr, a.X, a.dp, w.cp, w.cd, so.n);
        st.dist_evals = st.seed_evals = so.n;
        L = admit(w, cur, 0, so.n, sh.itopk);
        const uint32_t fan = sh.width * a.k_max;
        for (uint32_t it = 0; it < a.max_iter; ++it) {
          // frontier: first `width` unexpanded entries
          uint32_t nf = 0;
          for (uint32_t b0 = 0; b0 < L && nf < sh.width; b0 += 32) {
            uint32_t i = b0 + lane;
            bool un = i < L && w.qf[cur][i] == 0;
            uint32_t m = __ballot_sync(0xFFFFFFFFu, un);
            uint32_t rank = __popc(m & ((1u << lane) - 1));
            if (un && nf + rank < sh.width) {
              w.fr[nf + rank] = w.qp[cur][i];
              w.qf[cur][i] = 1;
            }
            nf = min(sh.width, nf + __popc(m));
          }
          __syncwarp();
          if (nf == 0) break;
          if (vis_n + nf * a.k_max > vcap) {
            overflow = true;
            break;
          }
          st.iterations++;
          st.expanded += nf;
          // gather, dedup, pre-check, visited
          clear_words(w.dedup, sh.dsz);
          __syncwarp();
          const uint32_t dlg = 31 - __clz(sh.dsz);
          uint32_t nc = 0;
          for (uint32_t b0 = 0; b0 < nf * a.k_max; b0 += 32) {
            uint32_t e = b0 + lane;
            bool cand = false, uniq = false, rej = false;
            uint32_t v = kSentinel, slot = 0;
            if (e < nf * a.k_max) {
              uint32_t row = w.fr[e / a.k_max];
              v = __ldg(a.adj + (uint64_t)row * a.k_max + (e % a.k_max));
              if (v != kSentinel) {
                Attr at = ld_attr(a.attr, v);
                slot = at.slot;
                if (slot < a.n_live) {
                  uniq = set_insert(w.dedup, dlg, v);
                  if (uniq) {
                    bool inr = at.s >= lo_f && at.s <= hi_f;
                    rej = !inr;
                    if (inr) cand = set_insert(w.vis, vlg, v);
                  }
                }
              }
            }
            uint32_t cm = __ballot_sync(0xFFFFFFFFu, cand);
            st.gathered += __popc(__ballot_sync(0xFFFFFFFFu, uniq));
            st.precheck_rejected += __popc(__ballot_sync(0xFFFFFFFFu, rej));
            if (cand) {
              uint32_t pos = nc + __popc(cm & ((1u << lane) - 1));
              w.cp[pos] = v;
              w.cs[pos] = slot;
            }
            nc += __popc(cm);
          }
          (void)fan;
          __syncwarp();
          vis_n += nc;
          if (nc == 0) continue;
          st.in_range_new += nc;
          st.dist_evals += nc;
          score<NC>(qr, a.X, a.dp, w.cp, w.cd, nc);
          L = admit(w, cur, L, nc, sh.itopk);
        }
      }
    }
    if (overflow) {
      if (lane == 0) {
        uint32_t pos = atomicAdd(a.ovf_count, 1u);
        a.ovf_list[pos] = qi;
      }
      continue;
    }
    const uint32_t cnt = min(L, a.k);
    for (uint32_t i = lane; i < a.k; i += 32) {
      a.out_slots[(uint64_t)qi * a.k + i] = i < cnt ? (int64_t)w.qs[cur][i] : -1;
      a.out_dists[(uint64_t)qi * a.k + i] = i < cnt ? w.qd[cur][i] : __longlong_as_double(0x7FF8000000000000ll);
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

static void launch(const SearchArgs& a, const SearchShape& sh, int num_sms, cudaStream_t st, uint32_t* gtab_ws,
                   uint32_t nwarps_cap) {
  const bool vis_smem = a.gtab == nullptr;
  const uint32_t wbytes = warp_smem_bytes(sh, vis_smem);
  uint32_t wpb = 4;
  while (wpb > 1 && wbytes * wpb > 200 * 1024) wpb >>= 1;
  const uint32_t smem = wbytes * wpb;
  if (smem > 227 * 1024) throw Error(GRAB_ERR_VALUE, "search parameters exceed shared memory (itopk too large)");
  uint32_t nc_chunks = (uint32_t)div_up(a.dp, 128);
  auto go = [&](auto kern) {
    GRAB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    GRAB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * wpb, smem));
    per_sm = per_sm < 1 ? 1 : per_sm;
    uint64_t blocks = div_up(a.nwork, wpb);
    uint64_t cap = (uint64_t)per_sm * num_sms;
    if (nwarps_cap) cap = std::min<uint64_t>(cap, div_up(nwarps_cap, wpb));
    blocks = std::min(blocks, cap);
    if (blocks == 0) return;
    kern<<<(unsigned)blocks, 32 * wpb, smem, st>>>(a, sh);
    GRAB_CHECK_LAUNCH();
  };
  if (nc_chunks <= 1)
    go(k_search<1>);
  else if (nc_chunks <= 2)
    go(k_search<2>);
  else if (nc_chunks <= 4)
    go(k_search<4>);
  else if (nc_chunks <= 8)
    go(k_search<8>);
  else
    throw Error(GRAB_ERR_VALUE, "dimension > 1024 not supported by the search kernel");
  (void)gtab_ws;
}

SearchShape make_shape(uint32_t itopk, uint32_t width, uint32_t k_max, uint32_t want, uint32_t max_iter, bool worst) {
  SearchShape s;
  s.itopk = itopk;
  s.width = width;
  uint32_t fan = width * k_max;
  s.cmax = 1u << ceil_log2(std::max<uint64_t>(std::max(fan, want), 32));  // bitonic pads to a power of 2
  s.dsz = 1u << ceil_log2(std::max<uint64_t>(2ull * fan, 128));
  if (!worst) {
    s.vlog2 = std::min<uint32_t>(14, std::max<uint32_t>(11, ceil_log2((uint64_t)itopk * 24)));
  } else {
    uint64_t bound = (uint64_t)want + (uint64_t)max_iter * fan + fan;
    s.vlog2 = std::max<uint32_t>(11, ceil_log2(bound * 4 / 3 + 1));
  }
  return s;
}

void run_search(const DevIndex& ix, SearchArgs a, cudaStream_t st) {
  if (a.nwork == 0) return;
  SearchShape sh = make_shape(a.itopk, a.width, a.k_max, a.want, a.max_iter, false);
  uint32_t* ovf;
  GRAB_CUDA(cudaMallocAsync(&ovf, (a.nwork + 1) * sizeof(uint32_t), st));
  GRAB_CUDA(cudaMemsetAsync(ovf, 0, sizeof(uint32_t), st));
  a.ovf_count = ovf;
  a.ovf_list = ovf + 1;
  a.gtab = nullptr;
  a.qmap = nullptr;
  launch(a, sh, ix.num_sms, st, nullptr, 0);
  uint32_t n_ovf = 0;
  GRAB_CUDA(cudaMemcpyAsync(&n_ovf, ovf, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
  GRAB_CUDA(cudaStreamSynchronize(st));
  if (n_ovf) {
    // exact re-run of the overflowed queries with a worst-case visited table
    SearchShape big = make_shape(a.itopk, a.width, a.k_max, a.want, a.max_iter, true);
    SearchArgs b = a;
    uint32_t* qmap;
    GRAB_CUDA(cudaMallocAsync(&qmap, n_ovf * sizeof(uint32_t), st));
    GRAB_CUDA(cudaMemcpyAsync(qmap, a.ovf_list, n_ovf * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st));
    b.qmap = qmap;
    b.nwork = n_ovf;
    GRAB_CUDA(cudaMemsetAsync(ovf, 0, sizeof(uint32_t), st));
    uint32_t nwarps = std::min<uint32_t>(n_ovf, 4u * (uint32_t)ix.num_sms);
    uint32_t* gtab = nullptr;
    if (warp_smem_bytes(big, true) > 200 * 1024) {
      uint64_t nwords = (uint64_t)nwarps * 4 * (1ull << big.vlog2);
      GRAB_CUDA(cudaMallocAsync(&gtab, nwords * 4, st));
      b.gtab = gtab;
    }
    launch(b, big, ix.num_sms, st, gtab, b.gtab ? nwarps : 0);
    uint32_t again = 0;
    GRAB_CUDA(cudaMemcpyAsync(&again, ovf, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    GRAB_CUDA(cudaStreamSynchronize(st));
    if (gtab) cudaFreeAsync(gtab, st);
    cudaFreeAsync(qmap, st);
    if (again) {
      cudaFreeAsync(ovf, st);
      throw Error(GRAB_ERR_CUDA, "visited-set overflow persisted on the worst-case retry");
    }
  }
  GRAB_CUDA(cudaFreeAsync(ovf, st));
}

}  // namespace grab
