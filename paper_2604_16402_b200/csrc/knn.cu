// kNN screen (f32 GEMM-expansion tiles + per-row max-heap of K + margin) and
// exact f64 rerank. Reference: pairwise_sq_dists / topk_ids_by_distance /
// exact_knn_graph (builder.py:79-127). The screen is a 128x128x32 SIMT tile
// GEMM with an in-CTA top-K' epilogue; the rerank recomputes each survivor
// with the library's f64 distance tree and applies the exact (dist, tiebreak)
// order, so the output equals the f64 oracle whenever the margin holds.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>

#include "knn.cuh"

namespace grab {

constexpr uint32_t BM = kKnnBM, BN = 128, BK = 32;
constexpr uint32_t kMargin = 16;
constexpr uint32_t kScreenTileBytes =
    (BK * (BM + 4) + BK * (BN + 4)) * 4 > BM * (BN + 1) * 4 ? (BK * (BM + 4) + BK * (BN + 4)) * 4 : BM * (BN + 1) * 4;

// Max-heap (h[0] largest) of one row, element i at h[i * BM]: rows are
// interleaved so neighbouring threads hit neighbouring banks.
// 4-ary (like the tcgen05 screen's): half the dependent load levels of a binary heap
__device__ __forceinline__ void heap_replace_top(uint64_t* h, uint32_t n, uint64_t key) {
  uint32_t i = 0;
  while (true) {
    const uint32_t c0 = 4 * i + 1;
    if (c0 >= n) break;
    uint64_t kb = h[c0 * BM];
    uint32_t big = c0;
#pragma unroll
    for (uint32_t j = 1; j < 4; ++j) {
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

__global__ void __launch_bounds__(256) k_knn_screen(const KnnJob* jobs, const float* X, const Attr* attr,
                                                    const float* norms, uint32_t dp, uint32_t KP, uint32_t* cand,
                                                    bool causal) {
  extern __shared__ __align__(16) uint8_t smem[];
  float* As = (float*)smem;                 // [BK][BM + 4]
  float* Bs = As + BK * (BM + 4);           // [BK][BN + 4]
  // the distance tile is written only after a column block's k-loop and read
  // before the next one starts (both fenced by __syncthreads), so it shares the
  // operand tiles' words -- room for K' up to ~150 heaps (insert at K_max 64)
  float* D = (float*)smem;                  // [BM][BN + 1]
  uint64_t* H = (uint64_t*)(smem + kScreenTileBytes);  // [BM][KP]
  const KnnJob job = jobs[blockIdx.x];
  const uint32_t t = threadIdx.x;
  const uint32_t ty = t >> 4, tx = t & 15;  // 16 x 16 threads, 8 x 8 outputs each
  for (uint32_t i = t; i < BM * KP; i += 256) H[i] = ~0ull;
  float a2[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    uint32_t r = ty * 8 + i;
    a2[i] = r < job.nr ? norms[job.r0 + r] : 0.f;
  }
  const uint32_t my_row = t < BM && t < job.nr ? job.r0 + t : kSentinel;
  __syncthreads();
  for (uint32_t cb = job.c0; cb < job.c1; cb += BN) {
    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
    for (uint32_t kb = 0; kb < dp; kb += BK) {
      // 128 rows x 32 cols per operand = 1024 float4; 4 per thread each
#pragma unroll
      for (int it = 0; it < 4; ++it) {
        uint32_t idx = t + 256 * it;
        uint32_t r = idx >> 3, k4 = (idx & 7) * 4;
        float4 va = make_float4(0, 0, 0, 0), vb = make_float4(0, 0, 0, 0);
        if (r < job.nr && kb + k4 < dp) va = *reinterpret_cast<const float4*>(X + (uint64_t)(job.r0 + r) * dp + kb + k4);
        if (cb + r < job.c1 && kb + k4 < dp) vb = *reinterpret_cast<const float4*>(X + (uint64_t)(cb + r) * dp + kb + k4);
        As[(k4 + 0) * (BM + 4) + r] = va.x;
        As[(k4 + 1) * (BM + 4) + r] = va.y;
        As[(k4 + 2) * (BM + 4) + r] = va.z;
        As[(k4 + 3) * (BM + 4) + r] = va.w;
        Bs[(k4 + 0) * (BN + 4) + r] = vb.x;
        Bs[(k4 + 1) * (BN + 4) + r] = vb.y;
        Bs[(k4 + 2) * (BN + 4) + r] = vb.z;
        Bs[(k4 + 3) * (BN + 4) + r] = vb.w;
      }
      __syncthreads();
#pragma unroll 8
      for (uint32_t k = 0; k < BK; ++k) {
        float4 a0 = *reinterpret_cast<const float4*>(As + k * (BM + 4) + ty * 8);
        float4 a1 = *reinterpret_cast<const float4*>(As + k * (BM + 4) + ty * 8 + 4);
        float4 b0 = *reinterpret_cast<const float4*>(Bs + k * (BN + 4) + tx * 8);
        float4 b1 = *reinterpret_cast<const float4*>(Bs + k * (BN + 4) + tx * 8 + 4);
        float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
        float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
      }
      __syncthreads();
    }
    // epilogue 1: distances into D (invalid -> +inf)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      uint32_t c = cb + tx * 8 + j;
      bool cv = c < job.c1 && attr[c].slot != kNoSlot;
      float b2 = cv ? norms[c] : 0.f;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        uint32_t r = ty * 8 + i;
        float d = fmaxf(a2[i] - 2.f * acc[i][j] + b2, 0.f);
        if (!cv || job.r0 + r == c || (causal && c > job.r0 + r)) d = __int_as_float(0x7F800000);
        D[r * (BN + 1) + tx * 8 + j] = d;
      }
    }
    __syncthreads();
    // epilogue 2: thread t < BM keeps row t's best KP by (screen dist, phys)
    if (my_row != kSentinel) {
      uint64_t* h = H + t;
      uint64_t top = h[0];
      const uint32_t ncol = min(BN, job.c1 - cb);
      for (uint32_t j = 0; j < ncol; ++j) {
        float d = D[t * (BN + 1) + j];
        uint64_t key = ((uint64_t)__float_as_uint(d) << 32) | (cb + j);
        if (key < top && d != __int_as_float(0x7F800000)) {
          heap_replace_top(h, KP, key);
          top = h[0];
        }
      }
    }
    __syncthreads();
  }
  if (my_row != kSentinel && attr[my_row].slot != kNoSlot) {
    uint64_t* h = H + t;
    for (uint32_t i = 0; i < KP; ++i)
      cand[(uint64_t)my_row * KP + i] = h[i * BM] == ~0ull ? kSentinel : (uint32_t)h[i * BM];
  }
}

// warp per row: f64 distances of the KP survivors, bitonic sort by
// (dist, tiebreak), keep K.
template <int NC>
__global__ void k_knn_rerank(const uint32_t* rows, uint64_t nrows, const uint32_t* cand, uint32_t KP, uint32_t P,
                             const float* X, const Attr* attr, uint32_t dp, uint32_t K, bool tb_slot,
                             uint32_t* out_ids, double* out_d) {
  extern __shared__ __align__(16) uint8_t smem[];
  const uint32_t wib = threadIdx.x >> 5, lane = lane_id(), wpb = blockDim.x >> 5;
  const uint64_t r = blockIdx.x * (uint64_t)wpb + wib;
  if (r >= nrows) return;
  double* sd = (double*)smem + wib * P;
  uint32_t* sk = (uint32_t*)((double*)smem + wpb * P) + wib * P;  // tiebreak
  uint32_t* sp = (uint32_t*)((double*)smem + wpb * P) + wpb * P + wib * P;  // phys
  const uint32_t p = rows[r];
  if (attr[p].slot == kNoSlot) return;
  float4 q[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    uint32_t col = (c * 32 + lane) * 4;
    q[c] = col < dp ? *reinterpret_cast<const float4*>(X + (uint64_t)p * dp + col) : make_float4(0, 0, 0, 0);
  }
  for (uint32_t i = lane; i < P; i += 32) {
    uint32_t c = i < KP ? cand[(uint64_t)p * KP + i] : kSentinel;
    sp[i] = c;
    sk[i] = c == kSentinel ? kSentinel : (tb_slot ? attr[c].slot : c);
    sd[i] = __longlong_as_double(0x7FF0000000000000ll);
  }
  __syncwarp();
  for (uint32_t i = 0; i < KP; ++i) {
    const uint32_t c = sp[i];
    if (c == kSentinel) continue;  // warp-uniform
    double acc = 0.0;
#pragma unroll
    for (int cc = 0; cc < NC; ++cc) {
      uint32_t col = (cc * 32 + lane) * 4;
      if (col < dp) acc = sq4(ldg_nc_f4(X + (uint64_t)c * dp + col), q[cc], acc);
    }
    acc = warp_sum(acc);
    if (lane == 0) sd[i] = acc;
  }
  __syncwarp();
  for (uint32_t k = 2; k <= P; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t i = lane; i < P; i += 32) {
        uint32_t l = i ^ j;
        if (l > i) {
          bool asc = (i & k) == 0;
          bool gt = key_less(sd[l], sk[l], sd[i], sk[i]);
          if (gt == asc) {
            double td = sd[i];
            sd[i] = sd[l];
            sd[l] = td;
            uint32_t tk = sk[i];
            sk[i] = sk[l];
            sk[l] = tk;
            uint32_t tp = sp[i];
            sp[i] = sp[l];
            sp[l] = tp;
          }
        }
      }
      __syncwarp();
    }
  }
  for (uint32_t i = lane; i < K; i += 32) {
    out_ids[(uint64_t)p * K + i] = sp[i];
    out_d[(uint64_t)p * K + i] = sd[i];
  }
}

void knn_device(const DevIndex& ix, const float* norms, const std::vector<KnnJob>& jobs, uint32_t K, bool tb_slot,
                uint32_t* out_ids, double* out_d, cudaStream_t st, bool causal) {
  if (jobs.empty()) return;
  const uint32_t KP = K + kMargin;
  uint32_t* cand;
  GRAB_CUDA(cudaMallocAsync(&cand, ix.phys_cap * (uint64_t)KP * 4, st));
  GRAB_CUDA(cudaMemsetAsync(cand, 0xFF, ix.phys_cap * (uint64_t)KP * 4, st));
  KnnJob* dj;
  GRAB_CUDA(cudaMallocAsync(&dj, jobs.size() * sizeof(KnnJob), st));
  GRAB_CUDA(cudaMemcpyAsync(dj, jobs.data(), jobs.size() * sizeof(KnnJob), cudaMemcpyHostToDevice, st));
  const bool dbg = getenv("GRAB_DEBUG") != nullptr;
  auto clk = [&]() {
    GRAB_CUDA(cudaStreamSynchronize(st));
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
  };
  const double t0 = dbg ? clk() : 0.0;
  const bool use_tc = knn_tc_supported(ix, KP);
  if (use_tc) {
    knn_screen_tc(ix, norms, dj, (uint32_t)jobs.size(), KP, cand, causal, st);
  } else {
    size_t smem = (size_t)kScreenTileBytes + (size_t)BM * KP * 8;
    if (smem > 227 * 1024) throw Error(GRAB_ERR_VALUE, "k too large for the kNN screen");
    GRAB_CUDA(cudaFuncSetAttribute(k_knn_screen, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_knn_screen<<<(unsigned)jobs.size(), 256, smem, st>>>(dj, ix.X, ix.attr, norms, ix.dp, KP, cand, causal);
    GRAB_CHECK_LAUNCH();
  }
  const double t1 = dbg ? clk() : 0.0;
  // rerank every row touched by a job
  std::vector<uint32_t> rows;
  for (const KnnJob& j : jobs)
    for (uint32_t i = 0; i < j.nr; ++i) rows.push_back(j.r0 + i);
  uint32_t* dr;
  GRAB_CUDA(cudaMallocAsync(&dr, rows.size() * 4, st));
  GRAB_CUDA(cudaMemcpyAsync(dr, rows.data(), rows.size() * 4, cudaMemcpyHostToDevice, st));
  uint32_t P = 32;
  while (P < KP) P <<= 1;
  const uint32_t wpb = 4;
  size_t rsmem = (size_t)wpb * P * 16;
  uint32_t nc = (uint32_t)div_up(ix.dp, 128);
  auto go = [&](auto kern) {
    GRAB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsmem));
    kern<<<(unsigned)div_up(rows.size(), wpb), 32 * wpb, rsmem, st>>>(dr, rows.size(), cand, KP, P, ix.X, ix.attr,
                                                                      ix.dp, K, tb_slot, out_ids, out_d);
    GRAB_CHECK_LAUNCH();
  };
  if (nc <= 1)
    go(k_knn_rerank<1>);
  else if (nc <= 2)
    go(k_knn_rerank<2>);
  else if (nc <= 4)
    go(k_knn_rerank<4>);
  else if (nc <= 8)
    go(k_knn_rerank<8>);
  else if (nc <= 16)
    go(k_knn_rerank<16>);
  else
    throw Error(GRAB_ERR_VALUE, "dimension > 2048 not supported");
  GRAB_CUDA(cudaStreamSynchronize(st));
  if (dbg) {
    const double t2 = clk();
    fprintf(stderr, "[grab] knn jobs=%zu K=%u %s screen %.3f s, rerank %.3f s\n", jobs.size(), K,
            use_tc ? "tcgen05" : "simt", t1 - t0, t2 - t1);
  }
  cudaFreeAsync(dr, st);
  cudaFreeAsync(dj, st);
  cudaFreeAsync(cand, st);
}

__global__ void k_norms(const float* X, uint64_t rows, uint32_t dp, float* out) {
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

void row_norms(const DevIndex& ix, float* out, cudaStream_t st) {
  if (!ix.phys_cap) return;
  k_norms<<<(unsigned)div_up(ix.phys_cap, 8), 256, 0, st>>>(ix.X, ix.phys_cap, ix.dp, out);
  GRAB_CHECK_LAUNCH();
}

}  // namespace grab
