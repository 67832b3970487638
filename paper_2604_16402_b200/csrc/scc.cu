// Strongly connected component count of the index graph on the device
// (reference evaluate.py:60-119, iterative Tarjan over the live rows).
//
// Tarjan is inherently sequential; the B200 restatement counts the same
// components with the coloring (forward-max / backward-closure) scheme:
//   repeat until no node is active:
//     trim: an active node with no active in-edge or no active out-edge is a
//           singleton SCC (counted, deactivated) -- iterated to a fixpoint;
//     color[v] = v, then propagate color[v] = max(color[v], color[u]) along
//           active edges u -> v to a fixpoint (edge-parallel sweeps);
//     every root (color[v] == v) owns exactly one SCC: the nodes of its color
//           that reach it -- marked by a backward closure restricted to the
//           color; count the roots, deactivate the marked nodes.
// Edges follow the reference's filter: SENTINEL and targets >= live_count are
// ignored (slot space; evaluate.py:71-73).
#include "index.cuh"

namespace grab {
namespace {

__global__ void k_scc_init(uint32_t n, const uint32_t* alive_in, uint8_t* active) {
  const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v < n) active[v] = alive_in ? (uint8_t)(alive_in[v] != 0) : 1;
}

// degree counts over active edges (trim)
__global__ void k_scc_deg(const uint32_t* adj, uint32_t n, uint32_t K, const uint8_t* active, uint32_t* indeg,
                          uint32_t* outdeg) {
  const uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (e >= (uint64_t)n * K) return;
  const uint32_t u = (uint32_t)(e / K), v = adj[e];
  if (v >= n || !active[u] || !active[v]) return;
  atomicAdd(indeg + v, 1u);
  atomicAdd(outdeg + u, 1u);
}

__global__ void k_scc_trim(uint32_t n, const uint32_t* indeg, const uint32_t* outdeg, uint8_t* active,
                           unsigned long long* count, uint32_t* changed) {
  const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n || !active[v]) return;
  if (indeg[v] == 0 || outdeg[v] == 0) {
    active[v] = 0;
    atomicAdd(count, 1ull);
    *changed = 1;
  }
}

__global__ void k_scc_color_init(uint32_t n, const uint8_t* active, uint32_t* color, uint8_t* mark) {
  const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n) return;
  color[v] = active[v] ? v : 0xFFFFFFFFu;
  mark[v] = 0;
}

__global__ void k_scc_fwd(const uint32_t* adj, uint32_t n, uint32_t K, const uint8_t* active, uint32_t* color,
                          uint32_t* changed) {
  const uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (e >= (uint64_t)n * K) return;
  const uint32_t u = (uint32_t)(e / K), v = adj[e];
  if (v >= n || !active[u] || !active[v]) return;
  const uint32_t cu = color[u];
  if (cu > color[v] && atomicMax(color + v, cu) < cu) *changed = 1;
}

__global__ void k_scc_roots(uint32_t n, const uint8_t* active, const uint32_t* color, uint8_t* mark,
                            unsigned long long* count) {
  const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v < n && active[v] && color[v] == v) {
    mark[v] = 1;
    atomicAdd(count, 1ull);
  }
}

// u -> v with v marked and the same color: u reaches the root too
__global__ void k_scc_bwd(const uint32_t* adj, uint32_t n, uint32_t K, const uint8_t* active, const uint32_t* color,
                          uint8_t* mark, uint32_t* changed) {
  const uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (e >= (uint64_t)n * K) return;
  const uint32_t u = (uint32_t)(e / K), v = adj[e];
  if (v >= n || !active[u] || mark[u] || !mark[v] || color[u] != color[v]) return;
  mark[u] = 1;
  *changed = 1;
}

__global__ void k_scc_retire(uint32_t n, uint8_t* active, const uint8_t* mark, uint32_t* left) {
  const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n || !active[v]) return;
  if (mark[v])
    active[v] = 0;
  else
    atomicAdd(left, 1u);
}

}  // namespace

// adj: slot-space rows [n x K] on the device (targets >= n / SENTINEL ignored)
uint64_t scc_count_device(const uint32_t* adj, uint32_t n, uint32_t K, cudaStream_t st) {
  if (n == 0) return 0;
  uint8_t *active, *mark;
  uint32_t *color, *indeg, *outdeg, *flag;
  unsigned long long* count;
  GRAB_CUDA(cudaMallocAsync(&active, n, st));
  GRAB_CUDA(cudaMallocAsync(&mark, n, st));
  GRAB_CUDA(cudaMallocAsync(&color, (size_t)n * 4, st));
  GRAB_CUDA(cudaMallocAsync(&indeg, (size_t)n * 4, st));
  GRAB_CUDA(cudaMallocAsync(&outdeg, (size_t)n * 4, st));
  GRAB_CUDA(cudaMallocAsync(&flag, 8, st));
  GRAB_CUDA(cudaMallocAsync(&count, 8, st));
  GRAB_CUDA(cudaMemsetAsync(count, 0, 8, st));
  const unsigned nb = (unsigned)div_up(n, 256);
  const unsigned eb = (unsigned)div_up((uint64_t)n * K, 256);
  k_scc_init<<<nb, 256, 0, st>>>(n, nullptr, active);
  auto read_flag = [&](uint32_t* f) {
    uint32_t h = 0;
    GRAB_CUDA(cudaMemcpyAsync(&h, f, 4, cudaMemcpyDeviceToHost, st));
    GRAB_CUDA(cudaStreamSynchronize(st));
    return h;
  };
  for (;;) {
    // trim to a fixpoint
    for (;;) {
      GRAB_CUDA(cudaMemsetAsync(indeg, 0, (size_t)n * 4, st));
      GRAB_CUDA(cudaMemsetAsync(outdeg, 0, (size_t)n * 4, st));
      GRAB_CUDA(cudaMemsetAsync(flag, 0, 4, st));
      k_scc_deg<<<eb, 256, 0, st>>>(adj, n, K, active, indeg, outdeg);
      k_scc_trim<<<nb, 256, 0, st>>>(n, indeg, outdeg, active, count, flag);
      GRAB_CHECK_LAUNCH();
      if (!read_flag(flag)) break;
    }
    k_scc_color_init<<<nb, 256, 0, st>>>(n, active, color, mark);
    for (;;) {
      GRAB_CUDA(cudaMemsetAsync(flag, 0, 4, st));
      k_scc_fwd<<<eb, 256, 0, st>>>(adj, n, K, active, color, flag);
      GRAB_CHECK_LAUNCH();
      if (!read_flag(flag)) break;
    }
    k_scc_roots<<<nb, 256, 0, st>>>(n, active, color, mark, count);
    for (;;) {
      GRAB_CUDA(cudaMemsetAsync(flag, 0, 4, st));
      k_scc_bwd<<<eb, 256, 0, st>>>(adj, n, K, active, color, mark, flag);
      GRAB_CHECK_LAUNCH();
      if (!read_flag(flag)) break;
    }
    GRAB_CUDA(cudaMemsetAsync(flag + 1, 0, 4, st));
    k_scc_retire<<<nb, 256, 0, st>>>(n, active, mark, flag + 1);
    GRAB_CHECK_LAUNCH();
    if (!read_flag(flag + 1)) break;
  }
  unsigned long long h = 0;
  GRAB_CUDA(cudaMemcpyAsync(&h, count, 8, cudaMemcpyDeviceToHost, st));
  GRAB_CUDA(cudaStreamSynchronize(st));
  for (void* p : {(void*)active, (void*)mark, (void*)color, (void*)indeg, (void*)outdeg, (void*)flag, (void*)count})
    cudaFreeAsync(p, st);
  return h;
}

}  // namespace grab
