// Two-pass static construction on the device (reference builder.py:503-548).
//
//   partition  (layout.py:107-154)   f32 radix sort -> quantile cuts / f32 linspace,
//                                      unique edges, bucket ids, stable slab layout
//   pass 1     (builder.py:189-261)  per-bucket exact kNN (screen + f64 rerank),
//                                      reverse lists by (dist, src), interleaved merge
//   pass 2     (builder.py:364-393)  exact global kNN (k_g) + reverse merge (338-361)
//   fuse       (builder.py:396-452)  proximal / global remote edges after the
//                                      necessary prefix, local fallback
//   repair     (builder.py:455-500)  sequential orphan repair, <= 4 rounds
//
// kNN is computed as a screen (f32 |a|^2 - 2ab + |b|^2 tiles, 2 x KP best per
// row) followed by an f64 rerank with the library's distance tree, so the
// selected lists equal the exact f64 (dist, tiebreak) top-k whenever the true
// top-k survives the screen (margin KP - k). The screen is the dense
// contraction; knn_tc.cu holds its tcgen05 tensor-core version.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <vector>

#include "index.cuh"
#include "knn.cuh"
#include "ops.cuh"

namespace grab {

static double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// ---------------------------------------------------------------- helpers
struct Scratch {
  std::vector<void*> ptrs;
  cudaStream_t st;
  explicit Scratch(cudaStream_t s) : st(s) {}
  template <class T>
  T* alloc(size_t n) {
    void* p = nullptr;
    GRAB_CUDA(cudaMallocAsync(&p, std::max<size_t>(n, 1) * sizeof(T), st));
    ptrs.push_back(p);
    return (T*)p;
  }
  ~Scratch() {
    for (void* p : ptrs) cudaFreeAsync(p, st);
  }
};

void exclusive_scan_u32(const uint32_t* in, uint32_t* out, uint64_t n, cudaStream_t st) {
  size_t tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, (int)n, st);
  void* t;
  GRAB_CUDA(cudaMallocAsync(&t, std::max<size_t>(tmp, 16), st));
  GRAB_CUDA(cub::DeviceScan::ExclusiveSum(t, tmp, in, out, (int)n, st));
  GRAB_CUDA(cudaFreeAsync(t, st));
}

__global__ void k_row_norms(const float* X, uint64_t rows, uint32_t dp, float* out) {
  uint64_t r = blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= rows) return;
  float acc = 0.f;
  for (uint32_t c = lane_id(); c < dp; c += 32) {
    float v = X[r * dp + c];
    acc = fmaf(v, v, acc);
  }
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, o);
  if (lane_id() == 0) out[r] = acc;
}

// ---------------------------------------------------------------- partition
__global__ void k_gather_cuts(const float* sorted, uint64_t n, const uint64_t* cuts, uint32_t m1, float* out) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m1) out[i] = sorted[cuts[i]];
}

__global__ void k_minmax(const float* s, uint64_t n, float* out /* [2] as ordered ints */) {
  float lo = INFINITY, hi = -INFINITY;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    lo = fminf(lo, s[i]);
    hi = fmaxf(hi, s[i]);
  }
  for (int o = 16; o; o >>= 1) {
    lo = fminf(lo, __shfl_xor_sync(0xFFFFFFFFu, lo, o));
    hi = fmaxf(hi, __shfl_xor_sync(0xFFFFFFFFu, hi, o));
  }
  if (lane_id() == 0) {
    // order-preserving int encoding of floats for atomicMin/Max
    auto enc = [](float f) {
      int b = __float_as_int(f);
      return b >= 0 ? b : b ^ 0x7FFFFFFF;
    };
    atomicMin((int*)out, enc(lo));
    atomicMax((int*)out + 1, enc(hi));
  }
}

static float dec_ordered(int b) { return b >= 0 ? *(float*)&b : [](int x) { x ^= 0x7FFFFFFF; return *(float*)&x; }(b); }

// Returns boundaries (host) per partition_buckets (layout.py:107-141).
std::vector<float> partition_edges_device(const float* S, uint64_t n, uint32_t target, int strategy,
                                          cudaStream_t st) {
  if (n < 1) throw Error(GRAB_ERR_VALUE, "cannot partition an empty scalar set");
  if (target < 1) throw Error(GRAB_ERR_VALUE, "target_capacity must be >= 1");
  uint64_t m = (n + target - 1) / target;
  std::vector<float> edges(m + 1);
  if (strategy == GRAB_STRATEGY_QUANTILE) {
    float* sorted;
    GRAB_CUDA(cudaMallocAsync(&sorted, n * 4, st));
    size_t tmp = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, tmp, S, sorted, (int)n, 0, 32, st);
    void* t;
    GRAB_CUDA(cudaMallocAsync(&t, std::max<size_t>(tmp, 16), st));
    GRAB_CUDA(cub::DeviceRadixSort::SortKeys(t, tmp, S, sorted, (int)n, 0, 32, st));
    std::vector<uint64_t> cuts(m + 1);
    const double step = (double)n / (double)m;
    for (uint64_t i = 0; i <= m; ++i) {
      double c = std::nearbyint((double)i * step);  // np.round: half to even
      cuts[i] = std::min<uint64_t>((uint64_t)c, n - 1);
    }
    cuts[m] = n - 1;
    uint64_t* dc;
    float* de;
    GRAB_CUDA(cudaMallocAsync(&dc, (m + 1) * 8, st));
    GRAB_CUDA(cudaMallocAsync(&de, (m + 1) * 4, st));
    GRAB_CUDA(cudaMemcpyAsync(dc, cuts.data(), (m + 1) * 8, cudaMemcpyHostToDevice, st));
    k_gather_cuts<<<(unsigned)div_up(m + 1, 256), 256, 0, st>>>(sorted, n, dc, (uint32_t)(m + 1), de);
    GRAB_CHECK_LAUNCH();
    GRAB_CUDA(cudaMemcpyAsync(edges.data(), de, (m + 1) * 4, cudaMemcpyDeviceToHost, st));
    GRAB_CUDA(cudaStreamSynchronize(st));
    cudaFreeAsync(dc, st);
    cudaFreeAsync(de, st);
    cudaFreeAsync(t, st);
    cudaFreeAsync(sorted, st);
  } else if (strategy == GRAB_STRATEGY_WIDTH) {
    int* mm;
    GRAB_CUDA(cudaMallocAsync(&mm, 8, st));
    int init[2] = {0x7FFFFFFF, (int)0x80000000};
    GRAB_CUDA(cudaMemcpyAsync(mm, init, 8, cudaMemcpyHostToDevice, st));
    k_minmax<<<256, 256, 0, st>>>(S, n, (float*)mm);
    GRAB_CHECK_LAUNCH();
    int h[2];
    GRAB_CUDA(cudaMemcpyAsync(h, mm, 8, cudaMemcpyDeviceToHost, st));
    GRAB_CUDA(cudaStreamSynchronize(st));
    cudaFreeAsync(mm, st);
    float lo = dec_ordered(h[0]), hi = dec_ordered(h[1]);
    // numpy evaluates linspace(f32 lo, f32 hi) in f32: step = (hi-lo)/m, y = i*step + lo
    volatile float delta = hi - lo;
    volatile float stepf = delta / (float)m;
    for (uint64_t i = 0; i <= m; ++i) {
      volatile float y = (float)i * stepf;
      edges[i] = y + lo;
    }
    edges[m] = hi;
  } else {
    throw Error(GRAB_ERR_VALUE, "unknown bucket strategy");
  }
  // np.unique on a non-decreasing sequence
  std::vector<float> u;
  for (float e : edges)
    if (u.empty() || e != u.back()) u.push_back(e);
  if (u.size() < 2) u = {u[0], u[0]};
  return u;
}

__global__ void k_hist(const int32_t* ids, uint64_t n, uint32_t* cnt) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i < n) atomicAdd(cnt + ids[i], 1u);
}

// ---------------------------------------------------------------- reverse CSR
// Given per-row forward lists fwd[r*K + j] (phys or SENTINEL) for rows
// [row0, row0 + nrows), build reverse CSR over target phys ids:
// rev_off[p] .. rev_off[p+1] hold (src phys, dist) for edges src->p.
__global__ void k_count_rev(const uint32_t* fwd, uint64_t nrows, uint32_t K, uint32_t* cnt) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= nrows * K) return;
  uint32_t v = fwd[i];
  if (v != kSentinel) atomicAdd(cnt + v, 1u);
}

__global__ void k_scatter_rev(const uint32_t* fwd, const double* fd, const uint32_t* rows, uint64_t nrows, uint32_t K,
                              const uint32_t* off, uint32_t* fill, uint32_t* rsrc, double* rdist) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= nrows * K) return;
  uint32_t v = fwd[i];
  if (v == kSentinel) return;
  uint32_t pos = off[v] + atomicAdd(fill + v, 1u);
  rsrc[pos] = rows[i / K];
  rdist[pos] = fd[i];
}

// ---------------------------------------------------------------- pass-1 merge
// warp per node: top-K_max of its reverse list by (dist, src phys), then the
// interleaved merge f0, r0, f1, r1, ... with dedup (builder.py:160-234).
__global__ void k_local_merge(const uint32_t* rows, uint64_t nrows, const uint32_t* fwd, uint32_t K,
                              const uint32_t* rev_off, const uint32_t* rsrc, const double* rdist, uint32_t k_local,
                              uint32_t* adj, uint32_t* necessary) {
  extern __shared__ __align__(16) uint8_t smem[];
  const uint32_t wib = threadIdx.x >> 5, lane = lane_id();
  const uint64_t r = blockIdx.x * (uint64_t)(blockDim.x >> 5) + wib;
  if (r >= nrows) return;
  double* ld = (double*)smem + wib * K;
  uint32_t* ls = (uint32_t*)((double*)smem + (blockDim.x >> 5) * K) + wib * K;
  const uint32_t p = rows[r];
  for (uint32_t i = lane; i < K; i += 32) {
    ld[i] = __longlong_as_double(0x7FF0000000000000ll);
    ls[i] = kSentinel;
  }
  __syncwarp();
  const uint32_t b = rev_off[p], e = rev_off[p + 1];
  for (uint32_t j = b; j < e; ++j) {  // warp-uniform loop
    const double d = rdist[j];
    const uint32_t s = rsrc[j];
    if (!key_less(d, s, ld[K - 1], ls[K - 1])) continue;
    uint32_t pos = 0;
    for (uint32_t b0 = 0; b0 < K; b0 += 32) {
      uint32_t i = b0 + lane;
      pos += __popc(__ballot_sync(0xFFFFFFFFu, i < K && key_less(ld[i], ls[i], d, s)));
    }
    for (int32_t hi = (int32_t)K - 1; hi > (int32_t)pos; hi -= 32) {
      int32_t i = hi - (int32_t)lane;
      bool mv = i > (int32_t)pos;
      double dv = mv ? ld[i - 1] : 0.0;
      uint32_t sv = mv ? ls[i - 1] : 0u;
      __syncwarp();
      if (mv) {
        ld[i] = dv;
        ls[i] = sv;
      }
      __syncwarp();
    }
    __syncwarp();  // every lane has read the list (no shift ran when pos == K - 1)
    if (lane == 0) {
      ld[pos] = d;
      ls[pos] = s;
    }
    __syncwarp();
  }
  // interleave; merged entries held one per lane (K <= 32 per chunk, K_max <= 64)
  uint32_t m0 = kSentinel, m1 = kSentinel;  // merged[lane], merged[32 + lane]
  uint32_t len = 0;
  const uint32_t* f = fwd + (uint64_t)p * K;
  for (uint32_t i = 0; i < K && len < K; ++i) {
    for (int src = 0; src < 2 && len < K; ++src) {
      uint32_t c = src == 0 ? f[i] : ls[i];
      if (c == kSentinel) continue;
      bool dup = __any_sync(0xFFFFFFFFu, (lane < len && m0 == c) || (32 + lane < len && m1 == c));
      if (dup) continue;
      if (len < 32) {
        if (lane == len) m0 = c;
      } else if (lane == len - 32) {
        m1 = c;
      }
      ++len;
    }
  }
  uint32_t* out = adj + (uint64_t)p * K;
  if (lane < K) out[lane] = lane < len ? m0 : kSentinel;
  if (32 + lane < K) out[32 + lane] = 32 + lane < len ? m1 : kSentinel;
  if (lane == 0) necessary[p] = min(len, k_local);
}

// ---------------------------------------------------------------- pass-2 union
// _reverse_merge_topk (builder.py:338-361): per node, union(forward, reverse),
// dedup, keep k_g by (dist, dst slot). Distances are the f64 kNN distances
// (symmetric, so the reverse edge reuses the forward edge's value).
__global__ void k_union_topk(const uint32_t* rows, uint64_t nrows, const uint32_t* fwd, const double* fd,
                             uint32_t K, const uint32_t* rev_off, const uint32_t* rsrc, const double* rdist,
                             const Attr* attr, uint32_t* G) {
  extern __shared__ __align__(16) uint8_t smem[];
  const uint32_t wib = threadIdx.x >> 5, lane = lane_id();
  const uint64_t r = blockIdx.x * (uint64_t)(blockDim.x >> 5) + wib;
  if (r >= nrows) return;
  double* ld = (double*)smem + wib * K;
  uint32_t* ls = (uint32_t*)((double*)smem + (blockDim.x >> 5) * K) + wib * K;  // slot key
  uint32_t* lp = ls + (blockDim.x >> 5) * K;                                      // phys
  const uint32_t p = rows[r];
  for (uint32_t i = lane; i < K; i += 32) {
    ld[i] = __longlong_as_double(0x7FF0000000000000ll);
    ls[i] = kSentinel;
    lp[i] = kSentinel;
  }
  __syncwarp();
  const uint32_t rb = rev_off[p], re = rev_off[p + 1];
  const uint32_t total = K + (re - rb);
  for (uint32_t j = 0; j < total; ++j) {
    uint32_t c;
    double d;
    if (j < K) {
      c = fwd[(uint64_t)p * K + j];
      if (c == kSentinel) continue;
      d = fd[(uint64_t)p * K + j];
    } else {
      c = rsrc[rb + j - K];
      d = rdist[rb + j - K];
    }
    const uint32_t s = attr[c].slot;
    if (!key_less(d, s, ld[K - 1], ls[K - 1])) continue;
    bool dup = false;
    uint32_t pos = 0;
    for (uint32_t b0 = 0; b0 < K; b0 += 32) {
      uint32_t i = b0 + lane;
      dup |= __any_sync(0xFFFFFFFFu, i < K && lp[i] == c);
      pos += __popc(__ballot_sync(0xFFFFFFFFu, i < K && key_less(ld[i], ls[i], d, s)));
    }
    if (dup) continue;
    for (int32_t hi = (int32_t)K - 1; hi > (int32_t)pos; hi -= 32) {
      int32_t i = hi - (int32_t)lane;
      bool mv = i > (int32_t)pos;
      double dv = mv ? ld[i - 1] : 0.0;
      uint32_t sv = mv ? ls[i - 1] : 0u, pv = mv ? lp[i - 1] : 0u;
      __syncwarp();
      if (mv) {
        ld[i] = dv;
        ls[i] = sv;
        lp[i] = pv;
      }
      __syncwarp();
    }
    __syncwarp();  // every lane has read the list (no shift ran when pos == K - 1)
    if (lane == 0) {
      ld[pos] = d;
      ls[pos] = s;
      lp[pos] = c;
    }
    __syncwarp();
  }
  for (uint32_t i = lane; i < K; i += 32) G[(uint64_t)p * K + i] = lp[i];
}

__global__ void k_iota(uint32_t* out, uint64_t n) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = (uint32_t)i;
}

// f64 distance of every edge (warp per row, the library's reduction tree);
// SENTINEL / self / out-of-range entries become SENTINEL
__global__ void k_edge_dists_f64(const float* X, uint32_t dp, uint64_t n, const uint32_t* g, uint32_t k,
                                 uint32_t* gf, double* gd) {
  const uint64_t v = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = lane_id();
  if (v >= n) return;
  for (uint32_t j = 0; j < k; ++j) {
    const uint32_t u = g[v * k + j];
    const bool ok = u != kSentinel && u < n && u != v;  // warp-uniform
    if (!ok) {
      if (lane == 0) gf[v * k + j] = kSentinel;
      continue;
    }
    double acc = 0.0;
    for (uint32_t col = lane * 4; col < dp; col += 128)
      acc = sq4(*reinterpret_cast<const float4*>(X + (uint64_t)u * dp + col),
                *reinterpret_cast<const float4*>(X + v * dp + col), acc);
    acc = warp_sum(acc);
    if (lane == 0) {
      gf[v * k + j] = u;
      gd[v * k + j] = acc;
    }
  }
}

__global__ void k_identity_attr(Attr* a, uint64_t n) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i < n) {
    a[i].s = 0.f;
    a[i].slot = (uint32_t)i;
  }
}

// _reverse_merge_topk (builder.py:338-361) over an explicit graph: the same
// reverse lists + union / dedup / top-k_g kernels the global pass runs (f64
// edge distances), on rows X[n x dim] with slot = row index. Host pointers.
void reverse_merge_raw(const float* X, uint64_t n, uint32_t dim, const uint32_t* graph, uint32_t k, uint32_t k_g,
                       uint32_t* out) {
  if (k > k_g) throw Error(GRAB_ERR_VALUE, "reverse merge: graph width above k_g");
  cudaStream_t st = 0;
  Scratch S(st);
  const uint32_t dp = (dim + 3) / 4 * 4;
  float* dX = S.alloc<float>(std::max<uint64_t>(n, 1) * dp);
  GRAB_CUDA(cudaMemsetAsync(dX, 0, std::max<uint64_t>(n, 1) * dp * 4, st));
  GRAB_CUDA(cudaMemcpy2DAsync(dX, dp * 4, X, dim * 4, dim * 4, n, cudaMemcpyHostToDevice, st));
  const uint64_t ne = n * (uint64_t)k;
  uint32_t* g = S.alloc<uint32_t>(std::max<uint64_t>(ne, 1));
  GRAB_CUDA(cudaMemcpyAsync(g, graph, ne * 4, cudaMemcpyHostToDevice, st));
  uint32_t* gf = S.alloc<uint32_t>(std::max<uint64_t>(ne, 1));
  double* gd = S.alloc<double>(std::max<uint64_t>(ne, 1));
  k_edge_dists_f64<<<(unsigned)div_up(n * 32, 256), 256, 0, st>>>(dX, dp, n, g, k, gf, gd);
  GRAB_CHECK_LAUNCH();
  Attr* attr = S.alloc<Attr>(std::max<uint64_t>(n, 1));
  k_identity_attr<<<(unsigned)div_up(n, 256), 256, 0, st>>>(attr, n);
  GRAB_CHECK_LAUNCH();
  uint32_t* cnt = S.alloc<uint32_t>(n + 1);
  uint32_t* off = S.alloc<uint32_t>(n + 1);
  uint32_t* fill = S.alloc<uint32_t>(std::max<uint64_t>(n, 1));
  uint32_t* prow = S.alloc<uint32_t>(std::max<uint64_t>(n, 1));
  k_iota<<<(unsigned)div_up(n, 256), 256, 0, st>>>(prow, n);
  GRAB_CHECK_LAUNCH();
  GRAB_CUDA(cudaMemsetAsync(cnt, 0, (n + 1) * 4, st));
  GRAB_CUDA(cudaMemsetAsync(fill, 0, n * 4, st));
  k_count_rev<<<(unsigned)div_up(ne, 256), 256, 0, st>>>(gf, n, k, cnt);
  GRAB_CHECK_LAUNCH();
  exclusive_scan_u32(cnt, off, n + 1, st);
  uint32_t nrev = 0;
  GRAB_CUDA(cudaMemcpyAsync(&nrev, off + n, 4, cudaMemcpyDeviceToHost, st));
  GRAB_CUDA(cudaStreamSynchronize(st));
  uint32_t* rsrc = S.alloc<uint32_t>(std::max<uint32_t>(nrev, 1));
  double* rdist = S.alloc<double>(std::max<uint32_t>(nrev, 1));
  k_scatter_rev<<<(unsigned)div_up(ne, 256), 256, 0, st>>>(gf, gd, prow, n, k, off, fill, rsrc, rdist);
  GRAB_CHECK_LAUNCH();
  // k_union_topk reads the forward rows with stride K = k_g: re-pack them
  uint32_t* gfk = S.alloc<uint32_t>(std::max<uint64_t>(n * (uint64_t)k_g, 1));
  double* gdk = S.alloc<double>(std::max<uint64_t>(n * (uint64_t)k_g, 1));
  GRAB_CUDA(cudaMemsetAsync(gfk, 0xFF, n * (uint64_t)k_g * 4, st));
  GRAB_CUDA(cudaMemcpy2DAsync(gfk, (size_t)k_g * 4, gf, (size_t)k * 4, (size_t)k * 4, n, cudaMemcpyDeviceToDevice, st));
  GRAB_CUDA(cudaMemcpy2DAsync(gdk, (size_t)k_g * 8, gd, (size_t)k * 8, (size_t)k * 8, n, cudaMemcpyDeviceToDevice, st));
  uint32_t* G = S.alloc<uint32_t>(std::max<uint64_t>(n * (uint64_t)k_g, 1));
  const uint32_t wpb = 4;
  const size_t smem = (size_t)wpb * k_g * 16;
  k_union_topk<<<(unsigned)div_up(n, wpb), 32 * wpb, smem, st>>>(prow, n, gfk, gdk, k_g, off, rsrc, rdist, attr, G);
  GRAB_CHECK_LAUNCH();
  GRAB_CUDA(cudaMemcpyAsync(out, G, n * (uint64_t)k_g * 4, cudaMemcpyDeviceToHost, st));
  GRAB_CUDA(cudaStreamSynchronize(st));
}

// ---------------------------------------------------------------- fuse
// fuse_remote_edges (builder.py:396-452); one thread per node.
__global__ void k_fuse(const uint32_t* rows, uint64_t nrows, const uint32_t* G, uint32_t k_g, const Attr* attr,
                       const int32_t* i2b, double window, uint32_t quota, uint32_t k_max, const uint32_t* necessary,
                       uint32_t* adj) {
  uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  const uint32_t p = rows[r];
  const Attr au = attr[p];
  const int32_t bu = i2b[au.slot];
  const double su = (double)au.s;
  const uint32_t start = necessary[p];
  const uint32_t room = k_max - start;
  // classify; count proximal picks (capped by quota) first
  uint32_t n_prox = 0;
  for (uint32_t j = 0; j < k_g; ++j) {
    uint32_t v = G[(uint64_t)p * k_g + j];
    if (v == kSentinel) continue;
    Attr av = attr[v];
    if (i2b[av.slot] == bu) continue;
    if (fabs((double)av.s - su) <= window && n_prox < quota) ++n_prox;
  }
  const int64_t budget = (int64_t)room - (int64_t)n_prox;
  uint32_t col = start;
  // proximal first (in G order), then global, each capped
  uint32_t taken_p = 0, taken_g = 0;
  for (int pass = 0; pass < 2; ++pass) {
    for (uint32_t j = 0; j < k_g; ++j) {
      uint32_t v = G[(uint64_t)p * k_g + j];
      if (v == kSentinel) continue;
      Attr av = attr[v];
      if (i2b[av.slot] == bu) continue;
      bool prox = fabs((double)av.s - su) <= window;
      if (pass == 0 && prox) {
        if (taken_p < quota) {
          ++taken_p;
          adj[(uint64_t)p * k_max + col++] = v;
        }
      } else if (pass == 1 && !prox) {
        if ((int64_t)(taken_g + 1) <= budget) {
          ++taken_g;
          adj[(uint64_t)p * k_max + col++] = v;
        }
      }
    }
  }
}

// ---------------------------------------------------------------- repair
__global__ void k_indegree(const uint32_t* adj, const uint32_t* rows, uint64_t nrows, uint32_t K, uint32_t* indeg) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= nrows * K) return;
  uint32_t v = adj[(uint64_t)rows[i / K] * K + i % K];
  if (v != kSentinel) atomicAdd(indeg + v, 1u);
}

// reinforce_reachability (builder.py:455-500): one warp walks the orphans in
// slot order; row distances via the library's f64 tree.
template <int NC>
__global__ void k_repair(const uint32_t* orphans, uint32_t n_orph, uint32_t* adj, uint32_t K, uint32_t k_local,
                         uint32_t* indeg, const float* X, uint32_t dp, uint32_t* added) {
  const uint32_t lane = lane_id();
  uint32_t n_added = 0;
  for (uint32_t t = 0; t < n_orph; ++t) {
    const uint32_t u = orphans[t];
    const uint32_t* ru = adj + (uint64_t)u * K;
    uint32_t v = kSentinel;
    for (uint32_t j = 0; j < K; ++j)
      if (ru[j] != kSentinel) {
        v = ru[j];
        break;
      }
    if (v == kSentinel) continue;
    uint32_t* row = adj + (uint64_t)v * K;
    int32_t free_pos = -1;
    for (uint32_t j = 0; j < K; ++j)
      if (row[j] == kSentinel) {
        free_pos = (int32_t)j;
        break;
      }
    if (free_pos >= 0) {
      if (lane == 0) row[free_pos] = u;
    } else {
      const uint32_t r0 = K > k_local ? k_local : 0;
      // distances d(v, row[j]) for the region; pick argmax among safe (indeg>=2) else region
      double best_safe = -1.0, best_any = -1.0;
      int32_t pos_safe = -1, pos_any = -1;
      float4 qv[NC];
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        uint32_t col = (c * 32 + lane) * 4;
        qv[c] = col < dp ? *reinterpret_cast<const float4*>(X + (uint64_t)v * dp + col) : make_float4(0, 0, 0, 0);
      }
      for (uint32_t j = r0; j < K; ++j) {
        const uint32_t w = row[j];
        double acc = 0.0;
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          uint32_t col = (c * 32 + lane) * 4;
          if (col < dp) acc = sq4(*reinterpret_cast<const float4*>(X + (uint64_t)w * dp + col), qv[c], acc);
        }
        acc = warp_sum(acc);
        if (acc > best_any) {
          best_any = acc;
          pos_any = (int32_t)j;
        }
        if (indeg[w] >= 2 && acc > best_safe) {
          best_safe = acc;
          pos_safe = (int32_t)j;
        }
      }
      const int32_t pos = pos_safe >= 0 ? pos_safe : pos_any;
      __syncwarp();
      if (lane == 0) {
        indeg[row[pos]] -= 1;
        row[pos] = u;
      }
    }
    __syncwarp();
    if (lane == 0) indeg[u] += 1;
    __syncwarp();
    ++n_added;
  }
  if (lane == 0) *added = n_added;
}

__global__ void k_cross_count(const uint32_t* adj, const uint32_t* rows, uint64_t nrows, uint32_t K, const Attr* attr,
                              const int32_t* i2b, unsigned long long* out) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  unsigned long long valid = 0, cross = 0;
  if (i < nrows * K) {
    uint32_t p = rows[i / K];
    uint32_t v = adj[(uint64_t)p * K + i % K];
    if (v != kSentinel) {
      valid = 1;
      cross = i2b[attr[v].slot] != i2b[attr[p].slot];
    }
  }
  for (int o = 16; o; o >>= 1) {
    valid += __shfl_xor_sync(0xFFFFFFFFu, valid, o);
    cross += __shfl_xor_sync(0xFFFFFFFFu, cross, o);
  }
  if (lane_id() == 0 && valid) {
    atomicAdd(out, valid);
    atomicAdd(out + 1, cross);
  }
}

__global__ void k_live_rows(const uint32_t* s2p, uint64_t n, uint32_t* rows) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i < n) rows[i] = s2p[i];
}

// phys-space rows -> slot-space host capture (debug / reference-shaped views)
__global__ void k_rows_to_slot(const uint32_t* src, uint32_t K, const uint32_t* s2p, const Attr* attr, uint64_t n,
                               uint32_t* out) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= n * K) return;
  uint32_t v = src[(uint64_t)s2p[i / K] * K + i % K];
  out[i] = v == kSentinel ? kSentinel : attr[v].slot;
}

static void capture_rows(const DevIndex& ix, const uint32_t* src, uint32_t K, uint64_t n, uint32_t* host,
                         cudaStream_t st) {
  if (!host || !n) return;
  uint32_t* tmp;
  GRAB_CUDA(cudaMallocAsync(&tmp, n * K * 4, st));
  k_rows_to_slot<<<(unsigned)div_up(n * K, 256), 256, 0, st>>>(src, K, ix.slot2phys, ix.attr, n, tmp);
  GRAB_CHECK_LAUNCH();
  GRAB_CUDA(cudaMemcpyAsync(host, tmp, n * K * 4, cudaMemcpyDeviceToHost, st));
  GRAB_CUDA(cudaStreamSynchronize(st));
  cudaFreeAsync(tmp, st);
}

__global__ void k_scatter_u32(const uint32_t* src, const uint32_t* s2p, uint64_t n, uint32_t* out) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i < n) out[s2p[i]] = src[i];
}

__global__ void k_gather_u32(const uint32_t* src, const uint32_t* s2p, uint64_t n, uint32_t* out) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = src[s2p[i]];
}

// ---------------------------------------------------------------- driver
static void launch_repair(const DevIndex& ix, const uint32_t* orph, uint32_t n, uint32_t* indeg, uint32_t* added,
                          cudaStream_t st) {
  uint32_t nc = (uint32_t)div_up(ix.dp, 128);
  const uint32_t K = ix.params.k_max, kl = ix.params.k_local;
  if (nc <= 1)
    k_repair<1><<<1, 32, 0, st>>>(orph, n, ix.adj, K, kl, indeg, ix.X, ix.dp, added);
  else if (nc <= 2)
    k_repair<2><<<1, 32, 0, st>>>(orph, n, ix.adj, K, kl, indeg, ix.X, ix.dp, added);
  else if (nc <= 4)
    k_repair<4><<<1, 32, 0, st>>>(orph, n, ix.adj, K, kl, indeg, ix.X, ix.dp, added);
  else if (nc <= 8)
    k_repair<8><<<1, 32, 0, st>>>(orph, n, ix.adj, K, kl, indeg, ix.X, ix.dp, added);
  else
    k_repair<16><<<1, 32, 0, st>>>(orph, n, ix.adj, K, kl, indeg, ix.X, ix.dp, added);
  GRAB_CHECK_LAUNCH();
}

__global__ void k_orphans(const uint32_t* indeg, const uint32_t* s2p, uint64_t n, uint32_t* list, uint32_t* cnt) {
  // slot order: one block scans a contiguous chunk; order restored by a sort on host side
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t p = s2p[i];
  if (indeg[p] == 0) {
    uint32_t pos = atomicAdd(cnt, 1u);
    list[pos] = (uint32_t)i;
  }
}

__global__ void k_slots_to_phys(uint32_t* list, uint32_t n, const uint32_t* s2p) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) list[i] = s2p[list[i]];
}

uint32_t reinforce_device(DevIndex& ix, const uint32_t* rows, uint64_t n, cudaStream_t st) {
  const uint32_t K = ix.params.k_max;
  Scratch S(st);
  uint32_t* indeg = S.alloc<uint32_t>(ix.phys_cap);
  uint32_t* list = S.alloc<uint32_t>(n);
  uint32_t* cnt = S.alloc<uint32_t>(2);
  uint32_t total = 0;
  for (int round = 0; round < 4; ++round) {
    GRAB_CUDA(cudaMemsetAsync(indeg, 0, ix.phys_cap * 4, st));
    GRAB_CUDA(cudaMemsetAsync(cnt, 0, 8, st));
    k_indegree<<<(unsigned)div_up(n * K, 256), 256, 0, st>>>(ix.adj, rows, n, K, indeg);
    GRAB_CHECK_LAUNCH();
    k_orphans<<<(unsigned)div_up(n, 256), 256, 0, st>>>(indeg, ix.slot2phys, n, list, cnt);
    GRAB_CHECK_LAUNCH();
    uint32_t no = 0;
    GRAB_CUDA(cudaMemcpyAsync(&no, cnt, 4, cudaMemcpyDeviceToHost, st));
    GRAB_CUDA(cudaStreamSynchronize(st));
    if (no == 0) break;
    // ascending slot order (np.flatnonzero), then to phys
    std::vector<uint32_t> h(no);
    GRAB_CUDA(cudaMemcpyAsync(h.data(), list, no * 4, cudaMemcpyDeviceToHost, st));
    GRAB_CUDA(cudaStreamSynchronize(st));
    std::sort(h.begin(), h.end());
    GRAB_CUDA(cudaMemcpyAsync(list, h.data(), no * 4, cudaMemcpyHostToDevice, st));
    k_slots_to_phys<<<(unsigned)div_up(no, 256), 256, 0, st>>>(list, no, ix.slot2phys);
    GRAB_CHECK_LAUNCH();
    launch_repair(ix, list, no, indeg, cnt + 1, st);
    uint32_t added = 0;
    GRAB_CUDA(cudaMemcpyAsync(&added, cnt + 1, 4, cudaMemcpyDeviceToHost, st));
    GRAB_CUDA(cudaStreamSynchronize(st));
    total += added;
  }
  return total;
}

constexpr uint64_t kExactGlobalLimit = 100000;  // EXACT_GLOBAL_LIMIT, builder.py:33
constexpr uint32_t kDescentSample = 8;            // descent_sample, builder.py:369
void descent_device(const DevIndex& ix, uint64_t n, uint32_t k, uint32_t rounds, uint32_t sample, uint32_t* gf,
                    double* gd, cudaStream_t st);  // descent.cu

void build_graph_device(DevIndex& ix, uint64_t n, uint32_t k_g, uint32_t refine_rounds, grab_build_report* rep,
                        const grab_build_debug* dbg, cudaStream_t st, uint32_t flags) {
  const uint32_t K = ix.params.k_max;
  const bool local_pass = !(flags & kGraphGlobalOnly), rest = !(flags & kGraphLocalOnly);
  Scratch S(st);
  uint32_t* rows = S.alloc<uint32_t>(n);  // phys rows in slot order
  k_live_rows<<<(unsigned)div_up(n, 256), 256, 0, st>>>(ix.slot2phys, n, rows);
  GRAB_CHECK_LAUNCH();
  float* norms = S.alloc<float>(ix.phys_cap);
  k_row_norms<<<(unsigned)div_up(ix.phys_cap, 8), 256, 0, st>>>(ix.X, ix.phys_cap, ix.dp, norms);
  GRAB_CHECK_LAUNCH();
  uint32_t* necessary = S.alloc<uint32_t>(ix.phys_cap);
  GRAB_CUDA(cudaMemsetAsync(necessary, 0, ix.phys_cap * 4, st));

  double t0 = now_s();
  // ---- pass 1: per-bucket kNN over slabs
  if (local_pass) {
  uint32_t* fwd = S.alloc<uint32_t>(ix.phys_cap * (uint64_t)K);
  double* fd = S.alloc<double>(ix.phys_cap * (uint64_t)K);
  {
    std::vector<KnnJob> jobs;
    uint32_t isolated = 0;
    for (uint32_t b = 0; b < ix.m; ++b) {
      uint32_t nb = ix.h_bcount[b], s0 = ix.h_bstart[b];
      if (nb == 1) ++isolated;
      if (nb < 2) continue;
      for (uint32_t r = 0; r < nb; r += kKnnBM) jobs.push_back({s0 + r, std::min<uint32_t>(kKnnBM, nb - r), s0, s0 + nb});
    }
    rep->isolated_nodes = isolated;
    GRAB_CUDA(cudaMemsetAsync(fwd, 0xFF, ix.phys_cap * (uint64_t)K * 4, st));
    knn_device(ix, norms, jobs, K, /*tiebreak slot=*/false, fwd, fd, st);
    if (dbg) capture_rows(ix, fwd, K, n, dbg->forward_rows, st);
  }
  // reverse lists + interleaved merge -> adjacency draft rows
  {
    uint32_t* cnt = S.alloc<uint32_t>(ix.phys_cap + 1);
    uint32_t* off = S.alloc<uint32_t>(ix.phys_cap + 1);
    uint32_t* fill = S.alloc<uint32_t>(ix.phys_cap);
    GRAB_CUDA(cudaMemsetAsync(cnt, 0, (ix.phys_cap + 1) * 4, st));
    GRAB_CUDA(cudaMemsetAsync(fill, 0, ix.phys_cap * 4, st));
    // fwd is indexed by phys row; iterate all phys rows (invalid rows are all-SENTINEL)
    uint32_t* prow = S.alloc<uint32_t>(ix.phys_cap);
    k_iota<<<(unsigned)div_up(ix.phys_cap, 256), 256, 0, st>>>(prow, ix.phys_cap);
    GRAB_CHECK_LAUNCH();
    uint64_t ne = ix.phys_cap * (uint64_t)K;
    k_count_rev<<<(unsigned)div_up(ne, 256), 256, 0, st>>>(fwd, ix.phys_cap, K, cnt);
    GRAB_CHECK_LAUNCH();
    exclusive_scan_u32(cnt, off, ix.phys_cap + 1, st);
    uint32_t nrev = 0;
    GRAB_CUDA(cudaMemcpyAsync(&nrev, off + ix.phys_cap, 4, cudaMemcpyDeviceToHost, st));
    GRAB_CUDA(cudaStreamSynchronize(st));
    uint32_t* rsrc = S.alloc<uint32_t>(nrev);
    double* rdist = S.alloc<double>(nrev);
    k_scatter_rev<<<(unsigned)div_up(ne, 256), 256, 0, st>>>(fwd, fd, prow, ix.phys_cap, K, off, fill, rsrc, rdist);
    GRAB_CHECK_LAUNCH();
    const uint32_t wpb = 4;
    size_t smem = (size_t)wpb * K * 12;
    k_local_merge<<<(unsigned)div_up(n, wpb), 32 * wpb, smem, st>>>(rows, n, fwd, K, off, rsrc, rdist,
                                                                    ix.params.k_local, ix.adj, necessary);
    GRAB_CHECK_LAUNCH();
  }
  GRAB_CUDA(cudaStreamSynchronize(st));
  if (dbg) {
    capture_rows(ix, ix.adj, K, n, dbg->merged_rows, st);
    if (dbg->necessary) {
      uint32_t* tmp;
      GRAB_CUDA(cudaMallocAsync(&tmp, n * 4, st));
      k_gather_u32<<<(unsigned)div_up(n, 256), 256, 0, st>>>(necessary, ix.slot2phys, n, tmp);
      GRAB_CHECK_LAUNCH();
      GRAB_CUDA(cudaMemcpyAsync(dbg->necessary, tmp, n * 4, cudaMemcpyDeviceToHost, st));
      GRAB_CUDA(cudaStreamSynchronize(st));
      cudaFreeAsync(tmp, st);
    }
  }
  }  // local_pass
  double t1 = now_s();
  if (!rest) {
    rep->phase1_seconds = t1 - t0;
    rep->total_seconds = t1 - t0;
    return;
  }

  // ---- pass 2: global kNN over all live rows, then reverse merge
  uint32_t* G = S.alloc<uint32_t>(ix.phys_cap * (uint64_t)k_g);
  GRAB_CUDA(cudaMemsetAsync(G, 0xFF, ix.phys_cap * (uint64_t)k_g * 4, st));
  if (n >= 2) {
    uint32_t* gf = S.alloc<uint32_t>(ix.phys_cap * (uint64_t)k_g);
    double* gd = S.alloc<double>(ix.phys_cap * (uint64_t)k_g);
    GRAB_CUDA(cudaMemsetAsync(gf, 0xFF, ix.phys_cap * (uint64_t)k_g * 4, st));
    // build_global_graph (builder.py:379-391): exact kNN at n <= EXACT_GLOBAL_LIMIT,
    // random init + neighborhood descent above (global_pass overrides)
    const uint32_t gp = ix.params.global_pass;
    const bool descent = gp == GRAB_GLOBAL_DESCENT || (gp == GRAB_GLOBAL_AUTO && n > kExactGlobalLimit);
    rep->global_descent = descent ? 1 : 0;
    if (descent) {
      descent_device(ix, n, k_g, refine_rounds, kDescentSample, gf, gd, st);
    } else {
      std::vector<KnnJob> jobs;
      const uint32_t pend = ix.h_bstart.back() + ix.h_bcount.back();
      for (uint32_t r = 0; r < pend; r += kKnnBM) jobs.push_back({r, std::min<uint32_t>(kKnnBM, pend - r), 0, pend});
      knn_device(ix, norms, jobs, k_g, /*tiebreak slot=*/true, gf, gd, st);
    }
    uint32_t* cnt = S.alloc<uint32_t>(ix.phys_cap + 1);
    uint32_t* off = S.alloc<uint32_t>(ix.phys_cap + 1);
    uint32_t* fill = S.alloc<uint32_t>(ix.phys_cap);
    uint32_t* prow = S.alloc<uint32_t>(ix.phys_cap);
    k_iota<<<(unsigned)div_up(ix.phys_cap, 256), 256, 0, st>>>(prow, ix.phys_cap);
    GRAB_CHECK_LAUNCH();
    GRAB_CUDA(cudaMemsetAsync(cnt, 0, (ix.phys_cap + 1) * 4, st));
    GRAB_CUDA(cudaMemsetAsync(fill, 0, ix.phys_cap * 4, st));
    uint64_t ne = ix.phys_cap * (uint64_t)k_g;
    k_count_rev<<<(unsigned)div_up(ne, 256), 256, 0, st>>>(gf, ix.phys_cap, k_g, cnt);
    GRAB_CHECK_LAUNCH();
    exclusive_scan_u32(cnt, off, ix.phys_cap + 1, st);
    uint32_t nrev = 0;
    GRAB_CUDA(cudaMemcpyAsync(&nrev, off + ix.phys_cap, 4, cudaMemcpyDeviceToHost, st));
    GRAB_CUDA(cudaStreamSynchronize(st));
    uint32_t* rsrc = S.alloc<uint32_t>(nrev);
    double* rdist = S.alloc<double>(nrev);
    k_scatter_rev<<<(unsigned)div_up(ne, 256), 256, 0, st>>>(gf, gd, prow, ix.phys_cap, k_g, off, fill, rsrc, rdist);
    GRAB_CHECK_LAUNCH();
    const uint32_t wpb = 4;
    size_t smem = (size_t)wpb * k_g * 16;
    k_union_topk<<<(unsigned)div_up(ix.phys_cap, wpb), 32 * wpb, smem, st>>>(prow, ix.phys_cap, gf, gd, k_g, off,
                                                                              rsrc, rdist, ix.attr, G);
    GRAB_CHECK_LAUNCH();
  }
  GRAB_CUDA(cudaStreamSynchronize(st));
  if (dbg) capture_rows(ix, G, k_g, n, dbg->global_rows, st);
  double t2 = now_s();
  if (!local_pass) {
    rep->phase2_seconds = t2 - t1;
    rep->total_seconds = t2 - t0;
    return;
  }

  // ---- fuse + repair
  {
    const double span = (double)ix.h_bound.back() - (double)ix.h_bound.front();
    const double window = ix.params.proximal_window * span;
    const double qf = ix.params.proximal_fraction * (double)(ix.params.k_max - ix.params.k_local);
    const uint32_t quota = (uint32_t)std::nearbyint(qf);  // Python round(): half to even
    if (n >= 2) {
      k_fuse<<<(unsigned)div_up(n, 256), 256, 0, st>>>(rows, n, G, k_g, ix.attr, ix.i2b, window, quota, K, necessary,
                                                       ix.adj);
      GRAB_CHECK_LAUNCH();
    }
    reinforce_device(ix, rows, n, st);
    unsigned long long* cc = S.alloc<unsigned long long>(2);
    GRAB_CUDA(cudaMemsetAsync(cc, 0, 16, st));
    k_cross_count<<<(unsigned)div_up(n * K, 256), 256, 0, st>>>(ix.adj, rows, n, K, ix.attr, ix.i2b, cc);
    GRAB_CHECK_LAUNCH();
    unsigned long long h[2];
    GRAB_CUDA(cudaMemcpyAsync(h, cc, 16, cudaMemcpyDeviceToHost, st));
    GRAB_CUDA(cudaStreamSynchronize(st));
    rep->cross_bucket_edge_ratio = h[0] ? (double)h[1] / (double)h[0] : 0.0;
  }
  double t3 = now_s();
  rep->phase1_seconds = t1 - t0;
  rep->phase2_seconds = t2 - t1;
  rep->fuse_seconds = t3 - t2;
  rep->total_seconds = t3 - t0;
}

// fuse_remote_edges (builder.py:396-452) over explicit inputs: the index's
// adjacency holds the draft rows (imported), `nec` / `G` are slot-space host
// arrays (necessary counts [n], global rows [n x k_g]).
__global__ void k_rows_slot_to_phys(const uint32_t* src, uint64_t n, uint32_t k, const uint32_t* s2p, uint32_t* dst) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= n * k) return;
  const uint32_t v = src[i];
  dst[(uint64_t)s2p[i / k] * k + i % k] = (v == kSentinel || v >= n) ? kSentinel : s2p[v];
}

void fuse_device(DevIndex& ix, uint64_t n, const uint32_t* nec_host, const uint32_t* G_host, uint32_t k_g) {
  cudaStream_t st = ix.stream;
  Scratch S(st);
  const uint32_t K = ix.params.k_max;
  uint32_t* rows = S.alloc<uint32_t>(n);
  k_live_rows<<<(unsigned)div_up(n, 256), 256, 0, st>>>(ix.slot2phys, n, rows);
  GRAB_CHECK_LAUNCH();
  uint32_t* nec_s = S.alloc<uint32_t>(n);
  uint32_t* nec = S.alloc<uint32_t>(ix.phys_cap);
  GRAB_CUDA(cudaMemsetAsync(nec, 0, ix.phys_cap * 4, st));
  GRAB_CUDA(cudaMemcpyAsync(nec_s, nec_host, n * 4, cudaMemcpyHostToDevice, st));
  k_scatter_u32<<<(unsigned)div_up(n, 256), 256, 0, st>>>(nec_s, ix.slot2phys, n, nec);
  GRAB_CHECK_LAUNCH();
  uint32_t* Gs = S.alloc<uint32_t>(n * (uint64_t)k_g);
  uint32_t* G = S.alloc<uint32_t>(ix.phys_cap * (uint64_t)k_g);
  GRAB_CUDA(cudaMemsetAsync(G, 0xFF, ix.phys_cap * (uint64_t)k_g * 4, st));
  GRAB_CUDA(cudaMemcpyAsync(Gs, G_host, n * (uint64_t)k_g * 4, cudaMemcpyHostToDevice, st));
  k_rows_slot_to_phys<<<(unsigned)div_up(n * k_g, 256), 256, 0, st>>>(Gs, n, k_g, ix.slot2phys, G);
  GRAB_CHECK_LAUNCH();
  const double span = (double)ix.h_bound.back() - (double)ix.h_bound.front();
  const double window = ix.params.proximal_window * span;
  const uint32_t quota = (uint32_t)std::nearbyint(ix.params.proximal_fraction * (double)(K - ix.params.k_local));
  k_fuse<<<(unsigned)div_up(n, 256), 256, 0, st>>>(rows, n, G, k_g, ix.attr, ix.i2b, window, quota, K, nec, ix.adj);
  GRAB_CHECK_LAUNCH();
  GRAB_CUDA(cudaStreamSynchronize(st));
}

uint32_t reinforce_index_device(DevIndex& ix) {
  cudaStream_t st = ix.stream;
  const uint64_t n = ix.count;
  if (!n) return 0;
  Scratch S(st);
  uint32_t* rows = S.alloc<uint32_t>(n);
  k_live_rows<<<(unsigned)div_up(n, 256), 256, 0, st>>>(ix.slot2phys, n, rows);
  GRAB_CHECK_LAUNCH();
  return reinforce_device(ix, rows, n, st);
}

void build_index_device(DevIndex& ix, const float* vectors, const float* scalars, uint64_t n, int strategy,
                        uint32_t k_g, uint32_t refine_rounds, uint32_t mem, grab_build_report* report,
                        const grab_build_debug* dbg) {
  cudaStream_t st = ix.stream;
  if (n < 1) throw Error(GRAB_ERR_VALUE, "cannot partition an empty scalar set");
  if (n > ix.n_cap) throw Error(GRAB_ERR_CAPACITY, "capacity exhausted: build of " + std::to_string(n) +
                                                       " rows > capacity " + std::to_string(ix.n_cap));
  if (k_g == 0) k_g = ix.params.k_max;
  Scratch S(st);
  const float* Xd = vectors;
  const float* Sd = scalars;
  if (mem == GRAB_MEM_HOST) {
    float* x = S.alloc<float>(n * ix.dim);
    float* s = S.alloc<float>(n);
    GRAB_CUDA(cudaMemcpyAsync(s, scalars, n * 4, cudaMemcpyHostToDevice, st));
    upload_h2d(x, vectors, n * ix.dim * 4, st);  // (pinned ring, parallel host copy)
    Xd = x;
    Sd = s;
    std::vector<float> hs(scalars, scalars + n);
    for (float v : hs)
      if (!std::isfinite(v)) throw Error(GRAB_ERR_VALUE, "scalars must be finite");
  }
  std::vector<float> edges = partition_edges_device(Sd, n, ix.params.bucket_capacity, strategy, st);
  ix.m = (uint32_t)edges.size() - 1;
  ix.h_bound = edges;
  ix.built = false;
  GRAB_CUDA(cudaMemsetAsync(ix.i2b, 0xFF, ix.n_cap * 4, st));
  {
    float* db = S.alloc<float>(edges.size());
    GRAB_CUDA(cudaMemcpyAsync(db, edges.data(), edges.size() * 4, cudaMemcpyHostToDevice, st));
    DevIndex tmp;
    tmp.bound = db;
    tmp.m = ix.m;
    launch_bucket_ids(tmp, Sd, n, ix.i2b, st);
  }
  uint32_t* hist = S.alloc<uint32_t>(ix.m);
  GRAB_CUDA(cudaMemsetAsync(hist, 0, ix.m * 4, st));
  k_hist<<<(unsigned)div_up(n, 256), 256, 0, st>>>(ix.i2b, n, hist);
  GRAB_CHECK_LAUNCH();
  std::vector<uint32_t> sizes(ix.m);
  GRAB_CUDA(cudaMemcpyAsync(sizes.data(), hist, ix.m * 4, cudaMemcpyDeviceToHost, st));
  GRAB_CUDA(cudaStreamSynchronize(st));
  layout_from_slots(ix, Xd, Sd, n, sizes);
  for (uint64_t i = 0; i < n; ++i) ix.ids[i] = (int64_t)i;
  grab_build_report rep{};
  rep.n = n;
  rep.m = ix.m;
  if (ix.params.k_max > 64) throw Error(GRAB_ERR_VALUE, "k_max > 64 not supported");
  build_graph_device(ix, n, k_g, refine_rounds, &rep, dbg, st, 0);
  ix.built = true;
  GRAB_CUDA(cudaStreamSynchronize(st));
  if (report) *report = rep;
}

}  // namespace grab
