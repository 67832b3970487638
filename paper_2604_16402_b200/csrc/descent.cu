// Pass-2 global graph above the exact limit: random init + neighborhood
// descent (reference builder.py:288-335, 364-393), on the device.
//
// Restated semantics (slot space, n nodes, k = k_g, s = descent_sample):
//   init    rng = default_rng([rng_seed, 1]);
//           graph = rng.integers(0, n - 1, size=(n, k)); graph[graph >= row] += 1
//           (numpy's bounded fill: Lemire 32-bit draws over a fill-local buffer
//           of the PCG64 stream, low half first) -- regenerated bit-exactly here
//           with 128-bit LCG jump-ahead, an accept scan and a scatter.
//   round   joint = [graph | reverse_topk(graph, dists, k)] (2k columns, the
//           reverse part = nearest k sources by (dist, src));
//           hop = rng.permutation(2k)[:2s] (numpy shuffle, bitgen-level 32-bit
//           buffer -- restated on the host);
//           candidates of v = joint[v] ++ joint[joint[v][h]] for h in hop (-1 if
//           missing); distance inf for missing, self and every repeat of an id
//           (first occurrence kept); new row = top-k by (dist, column).
// Distances are f64-accumulated then rounded to f32 (the reference's einsum
// accumulates in f32; values agree to the last bits, ids up to near-ties).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "index.cuh"
#include "rng.cuh"

namespace grab {

void exclusive_scan_u32(const uint32_t* in, uint32_t* out, uint64_t n, cudaStream_t st);  // build.cu

namespace {

struct ScratchD {
  std::vector<void*> ptrs;
  cudaStream_t st;
  explicit ScratchD(cudaStream_t s) : st(s) {}
  template <class T>
  T* alloc(size_t n) {
    void* p = nullptr;
    GRAB_CUDA(cudaMallocAsync(&p, std::max<size_t>(n, 1) * sizeof(T), st));
    ptrs.push_back(p);
    return (T*)p;
  }
  ~ScratchD() {
    for (void* p : ptrs) cudaFreeAsync(p, st);
  }
};

// (A, G) of a jump by m steps: s_m = A s + G inc.
struct Jump {
  u128 a, g;
};

__host__ __device__ inline Jump jump_compose(const Jump& x, const Jump& y) {  // x then y
  return Jump{y.a * x.a, y.a * x.g + y.g};
}

struct JumpPow2 {
  u128 a[64], g[64];
};

JumpPow2 make_pow2() {
  JumpPow2 t;
  Jump j{pcg_mult(), 1};
  for (int b = 0; b < 64; ++b) {
    t.a[b] = j.a;
    t.g[b] = j.g;
    j = jump_compose(j, j);
  }
  return t;
}

__host__ __device__ inline Jump jump_by(const u128* pa, const u128* pg, uint64_t m) {
  Jump acc{1, 0};
  for (int b = 0; m; ++b, m >>= 1)
    if (m & 1) acc = jump_compose(acc, Jump{pa[b], pg[b]});
  return acc;
}

// Host PCG64 with numpy's bitgen-level 32-bit buffer (pcg64_next32).
struct HostPcg {
  u128 state, inc;
  bool has32 = false;
  uint32_t buf32 = 0;
  uint64_t next64() {
    state = state * pcg_mult() + inc;
    return pcg_xsl_rr(state);
  }
  uint32_t next32() {
    if (has32) {
      has32 = false;
      return buf32;
    }
    const uint64_t x = next64();
    has32 = true;
    buf32 = (uint32_t)(x >> 32);
    return (uint32_t)x;
  }
  // random_interval(max): masked rejection over next32 (max < 2^32)
  uint32_t interval(uint32_t mx) {
    if (mx == 0) return 0;
    uint32_t mask = mx;
    mask |= mask >> 1;
    mask |= mask >> 2;
    mask |= mask >> 4;
    mask |= mask >> 8;
    mask |= mask >> 16;
    uint32_t v;
    while ((v = (next32() & mask)) > mx) {
    }
    return v;
  }
  // Generator.permutation(n): arange + Fisher-Yates from the top
  std::vector<uint32_t> permutation(uint32_t n) {
    std::vector<uint32_t> a(n);
    for (uint32_t i = 0; i < n; ++i) a[i] = i;
    for (uint32_t i = n - 1; i >= 1; --i) std::swap(a[i], a[interval(i)]);
    return a;
  }
};

// default_rng([a, b]) state (SeedSequence over two words)
Pcg64 pcg64_from_pair(uint64_t a, uint64_t b) {
  uint64_t e[2] = {a, b};
  SeedSeq s = seedseq_from_u64s(e, 2);
  uint64_t v[4];
  seedseq_u64(s, v, 4);
  const u128 initstate = ((u128)v[0] << 64) | v[1];
  const u128 initseq = ((u128)v[2] << 64) | v[3];
  Pcg64 g;
  g.inc = (initseq << 1) | 1;
  g.state = g.inc;
  g.state += initstate;
  g.state = g.state * pcg_mult() + g.inc;
  return g;
}

constexpr uint32_t kOutPerThread = 64;  // PCG outputs (128 words) per thread

// Word i of the stream (low/high halves of output i/2): Lemire accept flag and value.
__global__ void k_init_words(u128 s0, u128 inc, const u128* pa, const u128* pg, uint64_t n_out, uint32_t total,
                             uint32_t thresh, uint32_t* flag, uint32_t* val) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t o0 = t * kOutPerThread;
  if (o0 >= n_out) return;
  const Jump j = jump_by(pa, pg, o0);
  u128 s = j.a * s0 + j.g * inc;
  const uint64_t o1 = o0 + kOutPerThread < n_out ? o0 + kOutPerThread : n_out;
  for (uint64_t o = o0; o < o1; ++o) {
    s = s * pcg_mult() + inc;
    const uint64_t x = pcg_xsl_rr(s);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t w = (uint32_t)(x >> (32 * h));
      const uint64_t m = (uint64_t)w * total;
      flag[2 * o + h] = (uint32_t)m >= thresh ? 1u : 0u;
      val[2 * o + h] = (uint32_t)(m >> 32);
    }
  }
}

// graph[d] = value of the d-th accepted word (+1 when >= its row: no self)
__global__ void k_init_scatter(uint64_t n_words, const uint32_t* flag, const uint32_t* pos, const uint32_t* val,
                               uint64_t nk, uint32_t k, int32_t* graph, unsigned long long* last_word) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= n_words || !flag[i]) return;
  const uint64_t d = pos[i];
  if (d >= nk) return;
  const uint32_t row = (uint32_t)(d / k);
  uint32_t v = val[i];
  if (v >= row) v += 1;
  graph[d] = (int32_t)v;
  if (d == nk - 1) *last_word = i;
}

// f64-accumulated squared distance between slot rows a and b, rounded to f32;
// 8 lanes per pair (lane group g = lane / 8), dp/4 float4 per row.
__device__ __forceinline__ float group_dist(const float* X, uint32_t dp, uint32_t pa, uint32_t pb, uint32_t sub,
                                            bool active) {
  double acc = 0.0;
  if (active) {
    const float* ra = X + (uint64_t)pa * dp;
    const float* rb = X + (uint64_t)pb * dp;
    for (uint32_t f = sub; f * 4 < dp; f += 8) {
      const float4 x = ldg_nc_f4(rb + 4 * f);
      const float4 q = *reinterpret_cast<const float4*>(ra + 4 * f);
      acc = sq4(x, q, acc);
    }
  }
  acc += __shfl_xor_sync(0xFFFFFFFFu, acc, 4);
  acc += __shfl_xor_sync(0xFFFFFFFFu, acc, 2);
  acc += __shfl_xor_sync(0xFFFFFFFFu, acc, 1);
  return active ? (float)acc : __int_as_float(0x7F800000);
}

// init distances: one 8-lane group per edge
__global__ void k_edge_dists(const int32_t* graph, uint64_t nk, uint32_t k, const uint32_t* s2p, const float* X,
                             uint32_t dp, float* dist) {
  const uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = lane_id();
  const uint64_t e = w * 4 + lane / 8;
  const bool ok = e < nk && graph[e < nk ? e : 0] >= 0;
  const uint32_t row = (uint32_t)(e / k);
  const float d = group_dist(X, dp, ok ? s2p[row] : 0, ok ? s2p[graph[e]] : 0, lane & 7, ok);
  if (e < nk && (lane & 7) == 0) dist[e] = d;
}

// reverse top-k: key2 = (dist bits << 32 | src), sorted stably by dst afterwards
__global__ void k_rev_keys(const int32_t* graph, const float* dist, uint64_t nk, uint32_t k, uint32_t n,
                           uint64_t* key2, uint32_t* dst) {
  const uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (e >= nk) return;
  const int32_t v = graph[e];
  key2[e] = ((uint64_t)__float_as_uint(dist[e]) << 32) | (uint32_t)(e / k);
  dst[e] = v >= 0 ? (uint32_t)v : n;  // missing edges sort past every node
}

__global__ void k_count_dst(const uint32_t* dst, uint64_t nk, uint32_t n, uint32_t* cnt) {
  const uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (e < nk && dst[e] < n) atomicAdd(cnt + dst[e], 1u);
}

// joint[v] = [graph[v] (k) | nearest k reverse sources (-1 padded)], and
// jd[v] = their distances to v, already known: the forward ones from the
// current graph, the reverse ones from the reverse keys -- bit-identical to a
// recomputation (same lane-group order; (a-b)^2 == (b-a)^2 in f64)
__global__ void k_joint(const int32_t* graph, const float* dist, uint32_t n, uint32_t k, int32_t* joint, float* jd) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i < (uint64_t)n * k) {
    const uint64_t v = i / k, j = i % k;
    joint[v * 2 * k + j] = graph[i];
    joint[v * 2 * k + k + j] = -1;
    jd[v * 2 * k + j] = dist[i];
  }
}

__global__ void k_joint_rev(uint32_t n, uint32_t k, const uint32_t* sdst, const uint64_t* skey, const uint32_t* off,
                            uint64_t nk, int32_t* joint, float* jd) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= nk) return;
  const uint32_t v = sdst[i];
  if (v >= n) return;
  const uint64_t pos = i - off[v];
  if (pos < k) {
    joint[(uint64_t)v * 2 * k + k + pos] = (int32_t)(uint32_t)skey[i];
    jd[(uint64_t)v * 2 * k + k + pos] = __uint_as_float((uint32_t)(skey[i] >> 32));
  }
}

// Key of a (dist, column) candidate as one u64: f32 bits above the column.
__device__ __forceinline__ uint64_t dc_key(float d, uint32_t col) {
  return ((uint64_t)__float_as_uint(d) << 32) | col;
}

// One descent round: one warp per node. Shared memory per warp: candidate ids
// [C], a compute-flag bitmask [C/32] and an H-entry id hash. First occurrences are found in column order: chunk by
// chunk, the lowest lane of each id inside the chunk (match_any) inserts it,
// and an id already present from an earlier chunk is a repeat.
// jointp = the joint rows with every id mapped to its phys row (-1 kept), so
// candidate ids index X directly (no dependent slot -> phys load per row)
__global__ void k_joint_phys(const int32_t* joint, uint64_t total, const uint32_t* s2p, int32_t* jointp) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i < total) jointp[i] = joint[i] >= 0 ? (int32_t)s2p[joint[i]] : -1;
}

template <int WPB>
__global__ void __launch_bounds__(32 * WPB) k_descent(const int32_t* joint, const int32_t* jointp, uint32_t n,
                                                      uint32_t k, const uint32_t* hop, uint32_t nhop,
                                                      const uint32_t* s2p, const Attr* attr, const float* X,
                                                      uint32_t dp, uint32_t C, uint32_t H, int32_t* out_graph,
                                                      float* out_dist, const float* jd) {
  extern __shared__ __align__(16) uint8_t smem[];
  const uint32_t wib = threadIdx.x >> 5, lane = lane_id();
  const uint32_t v = blockIdx.x * WPB + wib;
  if (v >= n) return;  // warp-uniform
  const uint32_t NW = (C + 31) / 32;  // flag words
  uint8_t* base = smem + (size_t)wib * (C * 4 + NW * 4 + H * 2);
  int32_t* cid = (int32_t*)base;
  uint32_t* fl = (uint32_t*)(base + C * 4);  // bit i of word w: compute column 32 w + i
  // id hash of 16-bit entries = first column + 1 (the id itself is cid[entry - 1]):
  // half the shared memory of an id table, so more warps stay resident
  unsigned short* hkey = (unsigned short*)(fl + NW);
  const uint32_t J = 2 * k;
  const int32_t* jv = joint + (uint64_t)v * J;  // slot ids (hop sources index the joint rows)
  const uint32_t pv = s2p[v];
  // (a) candidate ids in PHYS space: own joint row, then the joint rows of the hop sources
  for (uint32_t i = lane; i < H / 2; i += 32) reinterpret_cast<uint32_t*>(hkey)[i] = 0u;
  for (uint32_t i = lane; i < J; i += 32) cid[i] = jointp[(uint64_t)v * J + i];
  for (uint32_t h = 0; h < nhop; ++h) {
    const int32_t src = jv[hop[h]];
    for (uint32_t i = lane; i < J; i += 32) cid[J + h * J + i] = src >= 0 ? jointp[(uint64_t)src * J + i] : -1;
  }
  __syncwarp();
  // (b) first occurrence per id, in column order
  const uint32_t hmask = H - 1;
  const float kInfF = __int_as_float(0x7F800000);
  for (uint32_t b0 = 0; b0 < C; b0 += 32) {
    const uint32_t c = b0 + lane;
    const int32_t id = c < C ? cid[c] : -1;
    const uint32_t same = __match_any_sync(0xFFFFFFFFu, (uint32_t)id);
    const bool lead = id >= 0 && (uint32_t)(__ffs(same) - 1) == lane;
    uint32_t h = ((uint32_t)id * 0x9E3779B1u) & hmask;
    const unsigned short me = (unsigned short)(c + 1);
    uint32_t cur = lead ? atomicCAS(hkey + h, (unsigned short)0, me) : 0u;
    bool pend = lead && cur != 0u && cid[cur - 1] != id;
    while (__any_sync(0xFFFFFFFFu, pend)) {
      if (pend) {
        h = (h + 1) & hmask;
        cur = atomicCAS(hkey + h, (unsigned short)0, me);
        pend = cur != 0u && cid[cur - 1] != id;
      }
    }
    const uint32_t m = __ballot_sync(0xFFFFFFFFu, lead && cur == 0u && (uint32_t)id != pv);
    if (lane == 0) fl[b0 >> 5] = m;
  }
  __syncwarp();
  // (c) distances of the first occurrences and (d) the running top-k by
  // (dist, column), 32 columns per chunk: 8-lane group g measures columns
  // c0 + 8g + u (u = 0..7, 4 rows in flight at a time); after the group's
  // xor-reduction lane 8g + s holds column c0 + 8g + s's distance in sums[s].
  const float* qrow = X + (uint64_t)pv * dp;
  const uint32_t sub = lane & 7, grp = lane >> 3;
  uint64_t best = ~0ull;  // lanes >= k never receive real entries
  for (uint32_t c0 = 0; c0 < C; c0 += 32) {
    const uint32_t flags = fl[c0 >> 5];
    if (c0 + 32 <= J) {
      // own joint row: every distance is known (no row loads)
      const uint32_t c = c0 + lane;
      uint64_t key = dc_key(((flags >> lane) & 1u) ? jd[(uint64_t)v * J + c] : kInfF, c);
      const uint64_t tail = __shfl_sync(0xFFFFFFFFu, best, k - 1);
      if (!__any_sync(0xFFFFFFFFu, key < tail)) continue;
      for (uint32_t kk = 2; kk <= 32; kk <<= 1)
        for (uint32_t j = kk >> 1; j > 0; j >>= 1) {
          const uint64_t o = __shfl_xor_sync(0xFFFFFFFFu, key, j);
          const bool up = (lane & kk) == 0, lower = (lane & j) == 0;
          if ((lower == up) ? (o < key) : (o > key)) key = o;
        }
      const uint64_t rev = __shfl_sync(0xFFFFFFFFu, key, 31 - lane);
      best = rev < best ? rev : best;
      for (uint32_t j = 16; j > 0; j >>= 1) {
        const uint64_t o = __shfl_xor_sync(0xFFFFFFFFu, best, j);
        const bool lower = (lane & j) == 0;
        if (lower ? (o < best) : (o > best)) best = o;
      }
      continue;
    }
    double sums[8];
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      uint32_t pc[4];
      bool ok[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t bit = grp * 8 + half * 4 + u;
        ok[u] = (flags >> bit) & 1u;
        pc[u] = ok[u] ? (uint32_t)cid[c0 + bit] : 0u;
      }
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 2
      for (uint32_t f = sub; f * 4 < dp; f += 8) {
        const float4 q = *reinterpret_cast<const float4*>(qrow + 4 * f);
        float4 x[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) x[u] = ok[u] ? ldg_nc_f4(X + (uint64_t)pc[u] * dp + 4 * f) : q;
#pragma unroll
        for (int u = 0; u < 4; ++u) acc[u] = sq4(x[u], q, acc[u]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        acc[u] += __shfl_xor_sync(0xFFFFFFFFu, acc[u], 4);
        acc[u] += __shfl_xor_sync(0xFFFFFFFFu, acc[u], 2);
        acc[u] += __shfl_xor_sync(0xFFFFFFFFu, acc[u], 1);
        sums[half * 4 + u] = acc[u];
      }
    }
    double mine = sums[0];
#pragma unroll
    for (int u = 1; u < 8; ++u) mine = sub == (uint32_t)u ? sums[u] : mine;
    const uint32_t c = c0 + lane;
    uint64_t key = c < C ? dc_key(((flags >> lane) & 1u) ? (float)mine : kInfF, c) : ~0ull;
    const uint64_t tail = __shfl_sync(0xFFFFFFFFu, best, k - 1);
    if (!__any_sync(0xFFFFFFFFu, key < tail)) continue;
    // sort the chunk ascending
    for (uint32_t kk = 2; kk <= 32; kk <<= 1)
      for (uint32_t j = kk >> 1; j > 0; j >>= 1) {
        const uint64_t o = __shfl_xor_sync(0xFFFFFFFFu, key, j);
        const bool up = (lane & kk) == 0, lower = (lane & j) == 0;
        if ((lower == up) ? (o < key) : (o > key)) key = o;
      }
    // merge: min(best[i], chunk[31 - i]) is bitonic and holds the 32 smallest
    const uint64_t rev = __shfl_sync(0xFFFFFFFFu, key, 31 - lane);
    best = rev < best ? rev : best;
    for (uint32_t j = 16; j > 0; j >>= 1) {
      const uint64_t o = __shfl_xor_sync(0xFFFFFFFFu, best, j);
      const bool lower = (lane & j) == 0;
      if (lower ? (o < best) : (o > best)) best = o;
    }
  }
  if (lane < k) {
    const uint32_t col = (uint32_t)best;
    const int32_t pid = cid[col];
    out_graph[(uint64_t)v * k + lane] = pid >= 0 ? (int32_t)attr[pid].slot : -1;
    out_dist[(uint64_t)v * k + lane] = __uint_as_float((uint32_t)(best >> 32));
  }
}

// ---------------------------------------------------------------- split round
// The same round in two phases, so a candidate row is read once per hop SOURCE
// instead of once per (node, candidate) pair. Node v's hop columns are the
// joint rows of u = joint[v][hop[h]]; every node that hops through u needs
// distances to the same J rows joint[u]. So:
//   A  (k_hop_dists) per source u: its J candidate rows and its users' rows
//      staged in shared memory, every (user, candidate) distance in f32 by
//      direct differences -- a screen value within g = dp * 2^-23 (relative)
//      of the exact squared distance -- written to buf[v][h][j];
//   B  (k_descent_split) per node: the same first-occurrence flags, then the
//      k-th smallest screen value T over flagged columns, then the EXACT
//      distance (group_dist: the direct round's arithmetic, bit for bit) for
//      every flagged column with screen value <= T (1 + 4 g'), g' >= g, and the
//      top k of those by (exact, column).
// Exactness: the k smallest screened columns have exact value <= T(1+g)(1+u),
// so the exact k-th is below that; a dropped column has exact value >=
// T(1+4g')(1-g)(1-u) > it, strictly, so it cannot be (or tie) a top-k entry.
// Own-row columns carry their exact distances already (jd), screen == exact.
constexpr uint32_t kHopUsers = 16, kHopPad = 132;  // users per chunk; smem row stride (floats)

// sources of every (v, h) pair: key = u (n for a missing column), value = v * nhop + h
__global__ void k_hop_pairs(const int32_t* joint, uint32_t n, uint32_t J, const uint32_t* hop, uint32_t nhop,
                            uint32_t* key, uint32_t* val) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= (uint64_t)n * nhop) return;
  const uint32_t v = (uint32_t)(i / nhop), h = (uint32_t)(i % nhop);
  const int32_t u = joint[(uint64_t)v * J + hop[h]];
  key[i] = u >= 0 ? (uint32_t)u : n;
  val[i] = (uint32_t)i;
}

__global__ void k_count_src(const uint32_t* key, uint64_t m, uint32_t n, uint32_t* cnt) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i < m && key[i] < n) atomicAdd(cnt + key[i], 1u);
}

// Packed FP32 pairs (Blackwell FADD2 / FFMA2): one instruction works on two
// dimensions, so the screen's even and odd dimensions accumulate in the two
// halves of a 64-bit register and are added at the end (a two-way split of the
// sum: its rounding bound is below the sequential one the margin `gam` covers).
__device__ __forceinline__ uint64_t f32x2_sub(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t f32x2_fma_sq(uint64_t d, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(r) : "l"(d), "l"(c));
  return r;
}
__device__ __forceinline__ float f32x2_hsum(uint64_t v) {
  return __uint_as_float((uint32_t)v) + __uint_as_float((uint32_t)(v >> 32));
}

// Block per source u (8 warps): warp w takes users 2w, 2w+1 of a 16-user chunk,
// lane l candidates l and l + 32; 128-float dimension chunks staged with a
// padded stride (conflict-free float4 reads).
__global__ void __launch_bounds__(256) k_hop_dists(const uint32_t* off, const uint32_t* sval, uint32_t n,
                                                   uint32_t nhop, uint32_t J, const int32_t* jointp,
                                                   const uint32_t* s2p, const float* X, uint32_t dp, float* buf) {
  __shared__ __align__(16) float cand[64 * kHopPad];
  __shared__ __align__(16) float usr[kHopUsers * kHopPad];
  __shared__ int32_t cph[64];
  __shared__ uint32_t uph[kHopUsers], upair[kHopUsers];
  const uint32_t u = blockIdx.x;
  const uint32_t b = off[u], e = off[u + 1];
  if (b == e) return;  // block-uniform
  const uint32_t tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  if (tid < 64) cph[tid] = tid < J ? jointp[(uint64_t)u * J + tid] : -1;
  const bool one_chunk = dp <= 128;
  auto load_cand = [&](uint32_t d0) {
    for (uint32_t i = tid; i < 64 * 32; i += 256) {
      const uint32_t r = i >> 5, c4 = (i & 31) * 4;
      float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
      const int32_t p = cph[r];
      if (p >= 0 && d0 + c4 < dp) x = ldg_nc_f4(X + (uint64_t)p * dp + d0 + c4);
      *reinterpret_cast<float4*>(cand + r * kHopPad + c4) = x;
    }
  };
  __syncthreads();
  if (one_chunk) load_cand(0);
  const uint32_t c0 = lane, c1 = lane + 32;
  for (uint32_t ub = b; ub < e; ub += kHopUsers) {
    const uint32_t nu = min(kHopUsers, e - ub);
    __syncthreads();  // the previous chunk's readers are done with usr / uph
    if (tid < kHopUsers) {
      const uint32_t pr = tid < nu ? sval[ub + tid] : 0u;
      upair[tid] = pr;
      uph[tid] = tid < nu ? s2p[pr / nhop] : 0u;
    }
    uint64_t acc[2][2] = {{0ull, 0ull}, {0ull, 0ull}};  // (even, odd) dimension partial sums
    for (uint32_t d0 = 0; d0 < dp; d0 += 128) {
      __syncthreads();
      if (!one_chunk) load_cand(d0);
      for (uint32_t i = tid; i < kHopUsers * 32; i += 256) {
        const uint32_t r = i >> 5, c4 = (i & 31) * 4;
        float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
        if (r < nu && d0 + c4 < dp) x = *reinterpret_cast<const float4*>(X + (uint64_t)uph[r] * dp + d0 + c4);
        *reinterpret_cast<float4*>(usr + r * kHopPad + c4) = x;
      }
      __syncthreads();
      const uint32_t dl = min(128u, dp - d0);
      const float* ca = cand + c0 * kHopPad;
      const float* cb = cand + c1 * kHopPad;
      const float* ua = usr + (2 * w) * kHopPad;
      const float* ubr = usr + (2 * w + 1) * kHopPad;
#pragma unroll 4
      for (uint32_t f = 0; f < dl; f += 4) {
        const ulonglong2 xa = *reinterpret_cast<const ulonglong2*>(ca + f);
        const ulonglong2 xb = *reinterpret_cast<const ulonglong2*>(cb + f);
        const ulonglong2 qa = *reinterpret_cast<const ulonglong2*>(ua + f);
        const ulonglong2 qb = *reinterpret_cast<const ulonglong2*>(ubr + f);
        const uint64_t xv[2][2] = {{xa.x, xa.y}, {xb.x, xb.y}};
        const uint64_t qv[2][2] = {{qa.x, qa.y}, {qb.x, qb.y}};
#pragma unroll
        for (int t = 0; t < 2; ++t)
#pragma unroll
          for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j) acc[i][j] = f32x2_fma_sq(f32x2_sub(xv[j][t], qv[i][t]), acc[i][j]);
      }
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const uint32_t ui = 2 * w + i;
      if (ui >= nu) continue;
      float* row = buf + (uint64_t)upair[ui] * J;  // pair index v * nhop + h
      const float kInfF = __int_as_float(0x7F800000);
      if (c0 < J) row[c0] = cph[c0] >= 0 ? f32x2_hsum(acc[i][0]) : kInfF;
      if (c1 < J) row[c1] = cph[c1] >= 0 ? f32x2_hsum(acc[i][1]) : kInfF;
    }
  }
}

// Phase B: one warp per node (see the split-round comment above).
template <int WPB>
__global__ void __launch_bounds__(32 * WPB) k_descent_split(const int32_t* joint, const int32_t* jointp, uint32_t n,
                                                            uint32_t k, const uint32_t* hop, uint32_t nhop,
                                                            const uint32_t* s2p, const Attr* attr, const float* X,
                                                            uint32_t dp, uint32_t C, uint32_t H, int32_t* out_graph,
                                                            float* out_dist, const float* jd, const float* buf,
                                                            double gam) {
  extern __shared__ __align__(16) uint8_t smem[];
  const uint32_t wib = threadIdx.x >> 5, lane = lane_id();
  const uint32_t v = blockIdx.x * WPB + wib;
  if (v >= n) return;  // warp-uniform
  const uint32_t NW = (C + 31) / 32;
  uint8_t* base = smem + (size_t)wib * (C * 4 + NW * 4 + H * 2);
  int32_t* cid = (int32_t*)base;
  uint32_t* fl = (uint32_t*)(base + C * 4);
  unsigned short* hkey = (unsigned short*)(fl + NW);
  unsigned short* rl = hkey;  // rerank list (columns): the id hash is dead once the flags are set (H >= C)
  const uint32_t J = 2 * k;
  const int32_t* jv = joint + (uint64_t)v * J;
  const uint32_t pv = s2p[v];
  // this node's screen values (nhop * J floats, contiguous) are read only after
  // the dedup: start pulling them into L2 now
  if (lane == 0) {
    const uint32_t bytes = nhop * J * 4;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(buf + (uint64_t)v * nhop * J), "r"(bytes)
                 : "memory");
  }
  // every hop source first (one load per lane), then all their id rows
  // back to back: the rows' loads are independent and overlap
  const int32_t src_l = lane < nhop ? jv[hop[lane]] : -1;
  for (uint32_t i = lane; i < H / 2; i += 32) reinterpret_cast<uint32_t*>(hkey)[i] = 0u;
  for (uint32_t i = lane; i < J; i += 32) cid[i] = jointp[(uint64_t)v * J + i];
#pragma unroll 4
  for (uint32_t h = 0; h < nhop; ++h) {
    const int32_t src = __shfl_sync(0xFFFFFFFFu, src_l, h);
    for (uint32_t i = lane; i < J; i += 32) cid[J + h * J + i] = src >= 0 ? jointp[(uint64_t)src * J + i] : -1;
  }
  __syncwarp();
  // first occurrence per id, in column order (k_descent's rule)
  const uint32_t hmask = H - 1;
  const float kInfF = __int_as_float(0x7F800000);
  for (uint32_t b0 = 0; b0 < C; b0 += 32) {
    const uint32_t c = b0 + lane;
    const int32_t id = c < C ? cid[c] : -1;
    const uint32_t same = __match_any_sync(0xFFFFFFFFu, (uint32_t)id);
    const bool lead = id >= 0 && (uint32_t)(__ffs(same) - 1) == lane;
    uint32_t h = ((uint32_t)id * 0x9E3779B1u) & hmask;
    const unsigned short me = (unsigned short)(c + 1);
    uint32_t cur = lead ? atomicCAS(hkey + h, (unsigned short)0, me) : 0u;
    bool pend = lead && cur != 0u && cid[cur - 1] != id;
    while (__any_sync(0xFFFFFFFFu, pend)) {
      if (pend) {
        h = (h + 1) & hmask;
        cur = atomicCAS(hkey + h, (unsigned short)0, me);
        pend = cur != 0u && cid[cur - 1] != id;
      }
    }
    const uint32_t m = __ballot_sync(0xFFFFFFFFu, lead && cur == 0u && (uint32_t)id != pv);
    if (lane == 0) fl[b0 >> 5] = m;
  }
  __syncwarp();
  const float* bv = buf + (uint64_t)v * nhop * J;  // screen values of the hop columns, in column order
  auto screen = [&](uint32_t c) -> float { return c < J ? jd[(uint64_t)v * J + c] : bv[c - J]; };
  // running top-k of 32-key chunks (k_descent's bitonic chunk merge)
  auto merge = [&](uint64_t& best, uint64_t key) {
    const uint64_t tail = __shfl_sync(0xFFFFFFFFu, best, k - 1);
    if (!__any_sync(0xFFFFFFFFu, key < tail)) return;
    for (uint32_t kk = 2; kk <= 32; kk <<= 1)
      for (uint32_t j = kk >> 1; j > 0; j >>= 1) {
        const uint64_t o = __shfl_xor_sync(0xFFFFFFFFu, key, j);
        const bool up = (lane & kk) == 0, lower = (lane & j) == 0;
        if ((lower == up) ? (o < key) : (o > key)) key = o;
      }
    const uint64_t rev = __shfl_sync(0xFFFFFFFFu, key, 31 - lane);
    best = rev < best ? rev : best;
    for (uint32_t j = 16; j > 0; j >>= 1) {
      const uint64_t o = __shfl_xor_sync(0xFFFFFFFFu, best, j);
      const bool lower = (lane & j) == 0;
      if (lower ? (o < best) : (o > best)) best = o;
    }
  };
  // (1) the k-th smallest screen value T over the flagged columns. The own
  // row's flagged columns are exact and contain at least k of them in the
  // common case, so their k-th smallest value Tu >= T bounds every column
  // that matters: only columns with screen value <= Tu (1 + 4g) are collected
  // (into rl) and ranked, instead of every one of the C columns.
  uint64_t obest = ~0ull;
  for (uint32_t c0 = 0; c0 < J; c0 += 32) {
    const uint32_t c = c0 + lane;
    const bool f = c < J && ((fl[c0 >> 5] >> lane) & 1u);
    merge(obest, f ? dc_key(jd[(uint64_t)v * J + c], c) : ~0ull);
  }
  const uint64_t tu = __shfl_sync(0xFFFFFFFFu, obest, k - 1);
  const double kInfD = __longlong_as_double(0x7FF0000000000000ll);
  const double ubound = tu == ~0ull ? kInfD : (double)__uint_as_float((uint32_t)(tu >> 32)) * (1.0 + 4.0 * gam);
  uint32_t nl = 0;
  for (uint32_t c0 = 0; c0 < C; c0 += 32) {
    const uint32_t c = c0 + lane;
    const bool take = c < C && ((fl[c0 >> 5] >> lane) & 1u) && (double)screen(c) <= ubound;
    const uint32_t m = __ballot_sync(0xFFFFFFFFu, take);
    if (take) rl[nl + __popc(m & ((1u << lane) - 1))] = (unsigned short)c;
    nl += __popc(m);
  }
  __syncwarp();
  uint64_t sbest = ~0ull;
  for (uint32_t i0 = 0; i0 < nl; i0 += 32) {
    const uint32_t i = i0 + lane;
    const uint32_t c = i < nl ? rl[i] : 0u;
    merge(sbest, i < nl ? dc_key(screen(c), c) : ~0ull);
  }
  const uint64_t tk = __shfl_sync(0xFFFFFFFFu, sbest, k - 1);
  const double bound = tk == ~0ull ? kInfD : (double)__uint_as_float((uint32_t)(tk >> 32)) * (1.0 + 4.0 * gam);
  // (2) columns that can still be in the top k (a subset of rl, kept in order)
  uint32_t nr = 0;
  for (uint32_t i0 = 0; i0 < nl; i0 += 32) {
    const uint32_t i = i0 + lane;
    const uint32_t c = i < nl ? rl[i] : 0u;
    const bool take = i < nl && (double)screen(c) <= bound;
    const uint32_t m = __ballot_sync(0xFFFFFFFFu, take);
    __syncwarp();  // the chunk is read before the compaction writes into it
    if (take) rl[nr + __popc(m & ((1u << lane) - 1))] = (unsigned short)c;
    nr += __popc(m);
  }
  __syncwarp();
  // (3) exact distances of those (own columns: jd; hop columns: group_dist in
  // k_descent's lane groups) and the top k by (exact, column)
  const float* qrow = X + (uint64_t)pv * dp;
  const uint32_t sub = lane & 7, grp = lane >> 3;
  uint64_t best = ~0ull;
  for (uint32_t r0 = 0; r0 < nr; r0 += 32) {
    double sums[8];
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      uint32_t pc[4];
      bool ok[4];
#pragma unroll
      for (int uu = 0; uu < 4; ++uu) {
        const uint32_t idx = r0 + grp * 8 + half * 4 + uu;
        const uint32_t c = idx < nr ? rl[idx] : 0u;
        ok[uu] = idx < nr && c >= J;
        pc[uu] = ok[uu] ? (uint32_t)cid[c] : 0u;
      }
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      if (__any_sync(0xFFFFFFFFu, ok[0] | ok[1] | ok[2] | ok[3])) {
#pragma unroll 2
        for (uint32_t f = sub; f * 4 < dp; f += 8) {
          const float4 q = *reinterpret_cast<const float4*>(qrow + 4 * f);
          float4 x[4];
#pragma unroll
          for (int uu = 0; uu < 4; ++uu) x[uu] = ok[uu] ? ldg_nc_f4(X + (uint64_t)pc[uu] * dp + 4 * f) : q;
#pragma unroll
          for (int uu = 0; uu < 4; ++uu) acc[uu] = sq4(x[uu], q, acc[uu]);
        }
      }
#pragma unroll
      for (int uu = 0; uu < 4; ++uu) {
        acc[uu] += __shfl_xor_sync(0xFFFFFFFFu, acc[uu], 4);
        acc[uu] += __shfl_xor_sync(0xFFFFFFFFu, acc[uu], 2);
        acc[uu] += __shfl_xor_sync(0xFFFFFFFFu, acc[uu], 1);
        sums[half * 4 + uu] = acc[uu];
      }
    }
    double mine = sums[0];
#pragma unroll
    for (int uu = 1; uu < 8; ++uu) mine = sub == (uint32_t)uu ? sums[uu] : mine;
    const uint32_t idx = r0 + lane;
    uint64_t key = ~0ull;
    if (idx < nr) {
      const uint32_t c = rl[idx];
      key = dc_key(c < J ? jd[(uint64_t)v * J + c] : (float)mine, c);
    }
    merge(best, key);
  }
  if (nr < k) {
    // fewer than k flagged columns: like k_descent, the rest of the row is the
    // (inf, column) keys of the unflagged columns, lowest columns first
    for (uint32_t c0 = 0; c0 < C; c0 += 32) {
      const uint32_t c = c0 + lane;
      const bool uf = c < C && !((fl[c0 >> 5] >> lane) & 1u);
      merge(best, uf ? dc_key(kInfF, c) : ~0ull);
    }
  }
  if (lane < k) {
    const uint32_t col = (uint32_t)best;
    const int32_t pid = best == ~0ull ? -1 : cid[col];
    out_graph[(uint64_t)v * k + lane] = pid >= 0 ? (int32_t)attr[pid].slot : -1;
    out_dist[(uint64_t)v * k + lane] = __uint_as_float((uint32_t)(best >> 32));
  }
}

// descent rows (slot ids) -> pass-2 forward rows in phys space with f64
// distances (the exact path's contract for the reverse merge)
__global__ void k_descent_to_phys(const int32_t* graph, uint32_t n, uint32_t k, const float* dist,
                                  const uint32_t* s2p, const float* X, uint32_t dp, uint32_t* gf, double* gd) {
  const uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = lane_id();
  if (w >= (uint64_t)n) return;
  const uint32_t v = (uint32_t)w, pv = s2p[v];
  // 8 edges per round, one f64 partial per edge per lane and reduce_scatter<8>
  // (the warp_sum tree, bit for bit): 4 rounds of loads in flight instead of 32
  // dependent ones
  constexpr int G = 8;
  for (uint32_t j0 = 0; j0 < k; j0 += G) {
    uint32_t pu[G];
    bool ok[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const uint32_t j = j0 + g;
      const int32_t u = j < k ? graph[(uint64_t)v * k + j] : -1;
      ok[g] = u >= 0 && (uint32_t)u != v && !isinf(dist[(uint64_t)v * k + j]);  // warp-uniform
      pu[g] = ok[g] ? s2p[u] : 0u;
    }
    double part[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      double acc = 0.0;
      if (ok[g])
        for (uint32_t col = lane * 4; col < dp; col += 128)
          acc = sq4(ldg_nc_f4(X + (uint64_t)pu[g] * dp + col),
                    *reinterpret_cast<const float4*>(X + (uint64_t)pv * dp + col), acc);
      part[g] = acc;
    }
    const double sum = reduce_scatter<G>(part);
    const uint32_t g = lane >> 2;  // lanes 4g .. 4g+3 hold edge j0 + g
    if ((lane & 3u) == 0 && j0 + g < k) {
      const uint32_t j = j0 + g;
      // (ok is warp-uniform per g; pick this lane's edge flags)
      bool okg = false;
      uint32_t pug = 0;
#pragma unroll
      for (int gg = 0; gg < G; ++gg)
        if ((uint32_t)gg == g) {
          okg = ok[gg];
          pug = pu[gg];
        }
      if (okg) {
        gf[(uint64_t)pv * k + j] = pug;
        gd[(uint64_t)pv * k + j] = sum;
      } else {
        gf[(uint64_t)pv * k + j] = kSentinel;
      }
    }
  }
}

}  // namespace

// Global NN-descent graph over slots [0, n): fills gf/gd (phys rows, phys ids,
// f64 distances, SENTINEL for unfilled) like knn_device does for the exact path.
void descent_device(const DevIndex& ix, uint64_t n64, uint32_t k, uint32_t rounds, uint32_t sample, uint32_t* gf,
                    double* gd, cudaStream_t st) {
  if (n64 < 3) throw Error(GRAB_ERR_VALUE, "descent needs at least 3 nodes");
  if (k > 32) throw Error(GRAB_ERR_VALUE, "descent supports k_g <= 32");
  if (n64 >= 0x7FFFFFFFull) throw Error(GRAB_ERR_VALUE, "descent supports n < 2^31");
  const uint32_t n = (uint32_t)n64;
  const uint64_t nk = (uint64_t)n * k;
  ScratchD S(st);
  // ---- init: graph = rng.integers(0, n - 1, (n, k)); += 1 where >= row
  const Pcg64 g0 = pcg64_from_pair(ix.params.rng_seed, 1);
  const JumpPow2 jt = make_pow2();
  u128* djt = S.alloc<u128>(128);
  GRAB_CUDA(cudaMemcpyAsync(djt, jt.a, sizeof(jt.a), cudaMemcpyHostToDevice, st));
  GRAB_CUDA(cudaMemcpyAsync(djt + 64, jt.g, sizeof(jt.g), cudaMemcpyHostToDevice, st));
  const uint32_t total = n - 1;                      // exclusive high n-1 -> values 0..n-2
  const uint32_t thresh = (uint32_t)((0x100000000ull - total) % total);
  int32_t* graph = S.alloc<int32_t>(nk);
  uint64_t consumed_out = 0;
  {
    uint64_t n_words = nk + nk / 64 + 4096;
    for (int attempt = 0;; ++attempt) {
      const uint64_t n_out = (n_words + 1) / 2;
      n_words = 2 * n_out;
      uint32_t* flag = S.alloc<uint32_t>(n_words + 1);
      uint32_t* val = S.alloc<uint32_t>(n_words);
      uint32_t* pos = S.alloc<uint32_t>(n_words + 1);
      unsigned long long* last = S.alloc<unsigned long long>(1);
      GRAB_CUDA(cudaMemsetAsync(last, 0xFF, 8, st));
      const uint64_t nthr = div_up(n_out, kOutPerThread);
      k_init_words<<<(unsigned)div_up(nthr, 128), 128, 0, st>>>(g0.state, g0.inc, djt, djt + 64, n_out, total,
                                                                thresh, flag, val);
      GRAB_CHECK_LAUNCH();
      GRAB_CUDA(cudaMemsetAsync(flag + n_words, 0, 4, st));
      exclusive_scan_u32(flag, pos, n_words + 1, st);
      uint32_t acc = 0;
      GRAB_CUDA(cudaMemcpyAsync(&acc, pos + n_words, 4, cudaMemcpyDeviceToHost, st));
      GRAB_CUDA(cudaStreamSynchronize(st));
      if (acc < nk) {
        if (attempt > 4) throw Error(GRAB_ERR_CUDA, "descent init: rejection stream too long");
        n_words = n_words * 2;
        continue;
      }
      k_init_scatter<<<(unsigned)div_up(n_words, 256), 256, 0, st>>>(n_words, flag, pos, val, nk, k, graph, last);
      GRAB_CHECK_LAUNCH();
      unsigned long long lw = 0;
      GRAB_CUDA(cudaMemcpyAsync(&lw, last, 8, cudaMemcpyDeviceToHost, st));
      GRAB_CUDA(cudaStreamSynchronize(st));
      consumed_out = (lw + 2) / 2;  // words 0..lw used -> ceil((lw + 1) / 2) outputs
      break;
    }
  }
  // generator state after the fill: the bitgen's own 32-bit buffer is untouched (empty)
  HostPcg hg;
  {
    const Jump j = jump_by(jt.a, jt.g, consumed_out);
    hg.state = j.a * g0.state + j.g * g0.inc;
    hg.inc = g0.inc;
  }
  float* dist = S.alloc<float>(nk);
  k_edge_dists<<<(unsigned)div_up(div_up(nk, 4) * 32, 256), 256, 0, st>>>(graph, nk, k, ix.slot2phys, ix.X, ix.dp,
                                                                         dist);
  GRAB_CHECK_LAUNCH();
  // ---- rounds
  const uint32_t s = std::min(sample, k);
  const uint32_t J = 2 * k, nhop = std::min(2 * s, J);
  const uint32_t C = J + nhop * J;
  uint32_t H = 1;
  while (H < C + C / 2) H <<= 1;  // id hash at load <= 2/3 (1088 candidates -> 2048)
  if (C >= 65535 || H > 65536) throw Error(GRAB_ERR_VALUE, "descent candidate set too large");
  int32_t* joint = S.alloc<int32_t>((uint64_t)n * J);
  int32_t* jointp = S.alloc<int32_t>((uint64_t)n * J);
  float* jd = S.alloc<float>((uint64_t)n * J);
  int32_t* g2 = S.alloc<int32_t>(nk);
  float* d2 = S.alloc<float>(nk);
  uint64_t* key2 = S.alloc<uint64_t>(nk);
  uint64_t* key2s = S.alloc<uint64_t>(nk);
  uint32_t* dst = S.alloc<uint32_t>(nk);
  uint32_t* dsts = S.alloc<uint32_t>(nk);
  uint64_t* key2t = S.alloc<uint64_t>(nk);
  uint32_t* dstt = S.alloc<uint32_t>(nk);
  uint32_t* cnt = S.alloc<uint32_t>(n + 1);
  uint32_t* off = S.alloc<uint32_t>(n + 1);
  uint32_t* dhop = S.alloc<uint32_t>(J);
  int end_bit = 1;
  while ((1ull << end_bit) <= n) ++end_bit;
  constexpr int WPB = 1;
  const size_t smem = (size_t)WPB * (C * 4 + (C + 31) / 32 * 4 + H * 2);
  GRAB_CUDA(cudaFuncSetAttribute(k_descent<WPB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  // split rounds (screen per hop source + exact rerank) while the per-node screen
  // buffer stays within budget; the direct kernel otherwise (and on request)
  const uint64_t npairs = (uint64_t)n * nhop;
  const bool split = !getenv("GRAB_DESCENT_DIRECT") && J <= 64 && npairs * J * 4 <= (12ull << 30) &&
                     npairs < 0xFFFFFFFFull;
  float* sbuf = nullptr;
  uint32_t *pkey = nullptr, *pval = nullptr, *pkeys = nullptr, *pvals = nullptr, *scnt = nullptr, *soff = nullptr;
  void* ptmp = nullptr;
  size_t ptmp_bytes = 0;
  const size_t smem_s = smem;  // (the rerank list aliases the id hash)
  // screen error bound: direct f32 differences, dp products summed in order
  const double gam = std::max(std::ldexp(1.0, -14), (double)ix.dp * std::ldexp(1.0, -22));
  if (split) {
    sbuf = S.alloc<float>(npairs * J);
    pkey = S.alloc<uint32_t>(npairs);
    pval = S.alloc<uint32_t>(npairs);
    pkeys = S.alloc<uint32_t>(npairs);
    pvals = S.alloc<uint32_t>(npairs);
    scnt = S.alloc<uint32_t>(n + 1);
    soff = S.alloc<uint32_t>(n + 1);
    cub::DeviceRadixSort::SortPairs(nullptr, ptmp_bytes, pkey, pkeys, pval, pvals, (int)npairs, 0, end_bit, st);
    ptmp = S.alloc<uint8_t>(ptmp_bytes);
    GRAB_CUDA(cudaFuncSetAttribute(k_descent_split<WPB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_s));
  }
  for (uint32_t r = 0; r < rounds; ++r) {
    // reverse top-k: stable sort by (dist, src), then by dst
    k_rev_keys<<<(unsigned)div_up(nk, 256), 256, 0, st>>>(graph, dist, nk, k, n, key2, dst);
    GRAB_CHECK_LAUNCH();
    size_t tmp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp, key2, key2s, dst, dstt, (int)nk, 0, 64, st);
    size_t tmp2 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp2, dstt, dsts, key2s, key2t, (int)nk, 0, end_bit, st);
    void* t = S.alloc<uint8_t>(std::max(tmp, tmp2));
    GRAB_CUDA(cub::DeviceRadixSort::SortPairs(t, tmp, key2, key2s, dst, dstt, (int)nk, 0, 64, st));
    GRAB_CUDA(cub::DeviceRadixSort::SortPairs(t, tmp2, dstt, dsts, key2s, key2t, (int)nk, 0, end_bit, st));
    GRAB_CUDA(cudaMemsetAsync(cnt, 0, (n + 1) * 4, st));
    k_count_dst<<<(unsigned)div_up(nk, 256), 256, 0, st>>>(dsts, nk, n, cnt);
    GRAB_CHECK_LAUNCH();
    exclusive_scan_u32(cnt, off, n + 1, st);
    k_joint<<<(unsigned)div_up(nk, 256), 256, 0, st>>>(graph, dist, n, k, joint, jd);
    GRAB_CHECK_LAUNCH();
    k_joint_rev<<<(unsigned)div_up(nk, 256), 256, 0, st>>>(n, k, dsts, key2t, off, nk, joint, jd);
    GRAB_CHECK_LAUNCH();
    const std::vector<uint32_t> perm = hg.permutation(J);
    GRAB_CUDA(cudaMemcpyAsync(dhop, perm.data(), nhop * 4, cudaMemcpyHostToDevice, st));
    k_joint_phys<<<(unsigned)div_up((uint64_t)n * J, 256), 256, 0, st>>>(joint, (uint64_t)n * J, ix.slot2phys, jointp);
    GRAB_CHECK_LAUNCH();
    if (split) {
      // users of every hop source (CSR by source), their screen distances, then the nodes
      k_hop_pairs<<<(unsigned)div_up(npairs, 256), 256, 0, st>>>(joint, n, J, dhop, nhop, pkey, pval);
      GRAB_CHECK_LAUNCH();
      GRAB_CUDA(cub::DeviceRadixSort::SortPairs(ptmp, ptmp_bytes, pkey, pkeys, pval, pvals, (int)npairs, 0, end_bit,
                                                st));
      GRAB_CUDA(cudaMemsetAsync(scnt, 0, (n + 1) * 4, st));
      k_count_src<<<(unsigned)div_up(npairs, 256), 256, 0, st>>>(pkeys, npairs, n, scnt);
      GRAB_CHECK_LAUNCH();
      exclusive_scan_u32(scnt, soff, n + 1, st);
      k_hop_dists<<<n, 256, 0, st>>>(soff, pvals, n, nhop, J, jointp, ix.slot2phys, ix.X, ix.dp, sbuf);
      GRAB_CHECK_LAUNCH();
      k_descent_split<WPB><<<(unsigned)div_up(n, WPB), 32 * WPB, smem_s, st>>>(
          joint, jointp, n, k, dhop, nhop, ix.slot2phys, ix.attr, ix.X, ix.dp, C, H, g2, d2, jd, sbuf, gam);
      GRAB_CHECK_LAUNCH();
    } else {
      k_descent<WPB><<<(unsigned)div_up(n, WPB), 32 * WPB, smem, st>>>(joint, jointp, n, k, dhop, nhop, ix.slot2phys,
                                                                       ix.attr, ix.X, ix.dp, C, H, g2, d2, jd);
      GRAB_CHECK_LAUNCH();
    }
    std::swap(graph, g2);
    std::swap(dist, d2);
    GRAB_CUDA(cudaStreamSynchronize(st));  // `perm` and the scratch stay valid across the round
  }
  k_descent_to_phys<<<(unsigned)div_up((uint64_t)n * 32, 256), 256, 0, st>>>(graph, n, k, dist, ix.slot2phys, ix.X,
                                                                            ix.dp, gf, gd);
  GRAB_CHECK_LAUNCH();
  GRAB_CUDA(cudaStreamSynchronize(st));
}

}  // namespace grab
