// Bucket-range sharded search: result packing and per-query top-k merge.
//
// The reference has no sharding (one process); this is the B200
// design for indexes split across GPUs by contiguous scalar (= bucket) range
// (SURVEY §8(e)): every rank searches only the queries whose range overlaps
// its shard, packs its per-query top-k -- mapped to GLOBAL slot ids -- into
// the block of the rank that owns the query, the blocks are exchanged with
// one fixed-size all-to-all (NCCL over NVLink), and each owner merges the
// world x k candidates of its queries by (distance, global slot), the
// reference's tie rule (searcher.py:64-71).
#include <algorithm>
#include <cstring>

#include "index.cuh"

namespace grab {

// send[(owner * B + q % B) * k + j] for every searched query q = qidx[i];
// blocks of unsearched queries keep the caller's 0xFF fill (NaN, -1).
__global__ void k_shard_pack(uint64_t n, const uint32_t* __restrict__ qidx, const int64_t* __restrict__ slots,
                             const double* __restrict__ dists, const int64_t* __restrict__ gid, uint32_t k,
                             uint32_t B, double* __restrict__ send_d, int64_t* __restrict__ send_i) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (t >= n * k) return;
  const uint64_t i = t / k, j = t % k;
  const uint32_t q = qidx[i];
  const uint64_t dst = ((uint64_t)(q / B) * B + q % B) * k + j;
  const int64_t s = slots[i * k + j];
  send_d[dst] = s >= 0 ? dists[i * k + j] : __longlong_as_double(0x7FF8000000000000ll);
  send_i[dst] = s >= 0 ? gid[s] : -1;
}

// One thread per owned query: k-way merge of nsrc ascending lists of k
// (entries with id < 0 are empty) into the top-k by (distance, global id).
__global__ void k_merge_topk(uint32_t nq, uint32_t nsrc, uint32_t B, uint32_t k, const double* __restrict__ d,
                             const int64_t* __restrict__ id, double* __restrict__ out_d, int64_t* __restrict__ out_i,
                             uint32_t* __restrict__ out_c) {
  const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  constexpr uint32_t kMaxSrc = 64;
  uint32_t head[kMaxSrc];
  for (uint32_t r = 0; r < nsrc; ++r) head[r] = 0;
  uint32_t c = 0;
  while (c < k) {
    int best = -1;
    double bd = 0;
    int64_t bi = 0;
    for (uint32_t r = 0; r < nsrc; ++r) {
      if (head[r] >= k) continue;
      const uint64_t o = ((uint64_t)r * B + q) * k + head[r];
      const int64_t ii = id[o];
      if (ii < 0) {
        head[r] = k;  // lists are dense prefixes
        continue;
      }
      const double dd = d[o];
      if (best < 0 || dd < bd || (dd == bd && ii < bi)) {
        best = (int)r;
        bd = dd;
        bi = ii;
      }
    }
    if (best < 0) break;
    out_d[(uint64_t)q * k + c] = bd;
    out_i[(uint64_t)q * k + c] = bi;
    head[best]++;
    ++c;
  }
  for (uint32_t j = c; j < k; ++j) {
    out_d[(uint64_t)q * k + j] = __longlong_as_double(0x7FF8000000000000ll);
    out_i[(uint64_t)q * k + j] = -1;
  }
  out_c[q] = c;
}

}  // namespace grab

using namespace grab;

extern "C" GRAB_API int grab_shard_pack(uint64_t n, const uint32_t* qidx, const int64_t* slots, const double* dists,
                                        const int64_t* gid, uint32_t k, uint32_t world, uint32_t B, double* send_d,
                                        int64_t* send_i, void* stream) {
  try {
    cudaStream_t st = (cudaStream_t)stream;
    if (k == 0 || world == 0 || B == 0) throw Error(GRAB_ERR_VALUE, "k, world and B must be >= 1");
    GRAB_CUDA(cudaMemsetAsync(send_d, 0xFF, (size_t)world * B * k * sizeof(double), st));
    GRAB_CUDA(cudaMemsetAsync(send_i, 0xFF, (size_t)world * B * k * sizeof(int64_t), st));
    if (n) {
      k_shard_pack<<<(unsigned)div_up(n * k, 256), 256, 0, st>>>(n, qidx, slots, dists, gid, k, B, send_d, send_i);
      GRAB_CHECK_LAUNCH();
    }
    return GRAB_OK;
  } catch (const Error& e) {
    return grab_set_error(e.code, e.what());
  }
}

extern "C" GRAB_API int grab_merge_topk(uint32_t nq, uint32_t nsrc, uint32_t B, uint32_t k, const double* d,
                                        const int64_t* id, double* out_d, int64_t* out_i, uint32_t* out_c,
                                        void* stream) {
  try {
    if (nsrc > 64) throw Error(GRAB_ERR_VALUE, "at most 64 shards");
    if (nq > B) throw Error(GRAB_ERR_VALUE, "owned queries exceed the block size");
    if (nq) {
      k_merge_topk<<<(unsigned)div_up(nq, 128), 128, 0, (cudaStream_t)stream>>>(nq, nsrc, B, k, d, id, out_d, out_i,
                                                                                out_c);
      GRAB_CHECK_LAUNCH();
    }
    return GRAB_OK;
  } catch (const Error& e) {
    return grab_set_error(e.code, e.what());
  }
}

// ---------------------------------------------------------------- peer-memory exchange
// The fused variant of pack + all-to-all: every rank stores its per-query
// top-k straight into the OWNER rank's receive buffer over NVLink (CUDA IPC
// mappings of the peers' buffers), so the exchange is the search epilogue's own
// stores -- no staging buffer, no collective kernel. recv layout on every rank:
// [src rank][B][k]; rank r writes only slice [r] of each owner's buffer.
namespace grab {

__global__ void k_shard_fill_p2p(uint64_t total, uint32_t rank, uint32_t B, uint32_t k, uint32_t world,
                                 double* const* peer_d, int64_t* const* peer_i) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (t >= total) return;  // total = world * B * k
  const uint32_t owner = (uint32_t)(t / ((uint64_t)B * k));
  const uint64_t within = t % ((uint64_t)B * k);
  const uint64_t off = (uint64_t)rank * B * k + within;
  peer_d[owner][off] = __longlong_as_double(0x7FF8000000000000ll);
  peer_i[owner][off] = -1;
}

__global__ void k_shard_pack_p2p(uint64_t n, const uint32_t* __restrict__ qidx, const int64_t* __restrict__ slots,
                                 const double* __restrict__ dists, const int64_t* __restrict__ gid, uint32_t k,
                                 uint32_t rank, uint32_t B, double* const* peer_d, int64_t* const* peer_i) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (t >= n * k) return;
  const uint64_t i = t / k, j = t % k;
  const uint32_t q = qidx[i];
  const uint32_t owner = q / B;
  const uint64_t off = ((uint64_t)rank * B + q % B) * k + j;
  const int64_t s = slots[i * k + j];
  peer_d[owner][off] = s >= 0 ? dists[i * k + j] : __longlong_as_double(0x7FF8000000000000ll);
  peer_i[owner][off] = s >= 0 ? gid[s] : -1;
  if (t == n * k - 1) __threadfence_system();
}

// ---- stream-ordered peer flags (no host round trip between pack and merge)
//
// Every rank owns one IPC-mapped sync block of u64 words: ready[world] (word s
// = the last batch epoch whose pack from rank s has fully landed in THIS
// rank's receive buffer) and free[world] (word r = the last epoch owner r has
// finished merging, so r's receive buffer may be overwritten), then a local
// completion counter. Per batch (epoch e, identical on every rank):
//   pack  (rank s): wait free[r] >= e - 1 for every owner r (its own block,
//         written remotely), write its whole slice of every owner's buffer,
//         last block: fence.sys, then ready[s] = e into every owner's block;
//   merge (owner r): wait ready[s] >= e for every s (its own block), merge,
//         last block: free[r] = e into every rank's block.
// All waits are device-side spins on system-scope acquire loads; the host
// enqueues search -> pack -> merge and never waits.
constexpr uint32_t kSyncReady = 0, kSyncCounter = 2;  // word offsets (x world for the first two)

__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// wait until words[0..world) >= target (one thread per block spins, then barrier)
__device__ __forceinline__ void wait_all_ge(const uint64_t* words, uint32_t world, uint64_t target) {
  if (threadIdx.x == 0) {
    for (uint32_t r = 0; r < world; ++r)
      while (ld_acquire_sys(words + r) < target) __nanosleep(200);
  }
  __syncthreads();
}

// true in exactly one thread of the grid: the last block to finish
__device__ __forceinline__ bool last_block(uint32_t* counter) {
  __shared__ bool last;
  __threadfence_system();  // this block's stores, before its arrival
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(counter, 1u) == gridDim.x - 1;
  __syncthreads();
  return last && threadIdx.x == 0;
}

__global__ void k_inv_map(uint64_t n, const uint32_t* qidx, int32_t* inv) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i < n) inv[qidx[i]] = (int32_t)i;
}

// Every entry of this rank's slice [rank][B][k] of every owner's buffer,
// exactly once: the packed top-k of a query this rank searched, else empty.
__global__ void k_shard_pack_p2p_sync(uint32_t nq, const int32_t* __restrict__ inv, const int64_t* __restrict__ slots,
                                      const double* __restrict__ dists, const int64_t* __restrict__ gid, uint32_t k,
                                      uint32_t rank, uint32_t world, uint32_t B, double* const* peer_d,
                                      int64_t* const* peer_i, uint64_t* my_sync, uint64_t* const* peer_sync,
                                      uint64_t epoch) {
  wait_all_ge(my_sync + (uint64_t)world, world, epoch - 1);  // every owner merged the previous batch
  const uint64_t total = (uint64_t)world * B * k;
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total; t += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t owner = (uint32_t)(t / ((uint64_t)B * k));
    const uint64_t within = t % ((uint64_t)B * k);
    const uint32_t ql = (uint32_t)(within / k), j = (uint32_t)(within % k);
    const uint32_t q = owner * B + ql;
    const int32_t i = q < nq ? inv[q] : -1;
    const int64_t s = i >= 0 ? slots[(uint64_t)i * k + j] : -1;
    const uint64_t off = (uint64_t)rank * B * k + within;
    peer_d[owner][off] = s >= 0 ? dists[(uint64_t)i * k + j] : __longlong_as_double(0x7FF8000000000000ll);
    peer_i[owner][off] = s >= 0 ? gid[s] : -1;
  }
  uint32_t* counter = reinterpret_cast<uint32_t*>(my_sync + (uint64_t)kSyncCounter * world);
  if (last_block(counter)) {
    *counter = 0;  // (stream order: the next pack starts after this kernel)
    for (uint32_t r = 0; r < world; ++r) st_release_sys(peer_sync[r] + kSyncReady * world + rank, epoch);
  }
}

__global__ void k_merge_topk_p2p(uint32_t nq, uint32_t nsrc, uint32_t B, uint32_t k, const double* __restrict__ d,
                                 const int64_t* __restrict__ id, double* __restrict__ out_d,
                                 int64_t* __restrict__ out_i, uint32_t* __restrict__ out_c, uint32_t rank,
                                 uint64_t* my_sync, uint64_t* const* peer_sync, uint64_t epoch) {
  wait_all_ge(my_sync + kSyncReady * nsrc, nsrc, epoch);  // every rank's slice has landed
  const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q < nq) {
    uint32_t head[64];
    for (uint32_t r = 0; r < nsrc; ++r) head[r] = 0;
    uint32_t c = 0;
    while (c < k) {
      int best = -1;
      double bd = 0;
      int64_t bi = 0;
      for (uint32_t r = 0; r < nsrc; ++r) {
        if (head[r] >= k) continue;
        const uint64_t o = ((uint64_t)r * B + q) * k + head[r];
        const int64_t ii = id[o];
        if (ii < 0) {
          head[r] = k;
          continue;
        }
        const double dd = d[o];
        if (best < 0 || dd < bd || (dd == bd && ii < bi)) {
          best = (int)r;
          bd = dd;
          bi = ii;
        }
      }
      if (best < 0) break;
      out_d[(uint64_t)q * k + c] = bd;
      out_i[(uint64_t)q * k + c] = bi;
      head[best]++;
      c++;
    }
    for (uint32_t j = c; j < k; ++j) {
      out_d[(uint64_t)q * k + j] = __longlong_as_double(0x7FF8000000000000ll);
      out_i[(uint64_t)q * k + j] = -1;
    }
    out_c[q] = c;
  }
  uint32_t* counter = reinterpret_cast<uint32_t*>(my_sync + (uint64_t)kSyncCounter * nsrc) + 1;
  if (last_block(counter)) {
    *counter = 0;
    for (uint32_t s = 0; s < nsrc; ++s) st_release_sys(peer_sync[s] + (uint64_t)nsrc + rank, epoch);
  }
}

}  // namespace grab

extern "C" GRAB_API uint64_t grab_shard_sync_bytes(uint32_t world) { return (uint64_t)(2 * world + 1) * 8; }

extern "C" GRAB_API int grab_shard_pack_p2p_sync(uint32_t nq, uint64_t n, const uint32_t* qidx, const int64_t* slots,
                                                 const double* dists, const int64_t* gid, uint32_t k, uint32_t rank,
                                                 uint32_t world, uint32_t B, double* const* peer_d,
                                                 int64_t* const* peer_i, uint64_t* my_sync,
                                                 uint64_t* const* peer_sync, uint64_t epoch, int32_t* inv_scratch,
                                                 void* stream) {
  try {
    cudaStream_t st = (cudaStream_t)stream;
    if (k == 0 || world == 0 || B == 0 || rank >= world || epoch == 0) throw Error(GRAB_ERR_VALUE, "bad shard geometry");
    if ((uint64_t)B * world < nq) throw Error(GRAB_ERR_VALUE, "owner blocks do not cover the batch");
    GRAB_CUDA(cudaMemsetAsync(inv_scratch, 0xFF, (size_t)std::max<uint32_t>(nq, 1) * 4, st));
    if (n) {
      k_inv_map<<<(unsigned)div_up(n, 256), 256, 0, st>>>(n, qidx, inv_scratch);
      GRAB_CHECK_LAUNCH();
    }
    const uint64_t total = (uint64_t)world * B * k;
    const unsigned blocks = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(div_up(total, 256), 1024));
    k_shard_pack_p2p_sync<<<blocks, 256, 0, st>>>(nq, inv_scratch, slots, dists, gid, k, rank, world, B, peer_d,
                                                   peer_i, my_sync, peer_sync, epoch);
    GRAB_CHECK_LAUNCH();
    return GRAB_OK;
  } catch (const Error& e) {
    return grab_set_error(e.code, e.what());
  }
}

extern "C" GRAB_API int grab_merge_topk_p2p(uint32_t nq, uint32_t nsrc, uint32_t B, uint32_t k, const double* d,
                                           const int64_t* id, double* out_d, int64_t* out_i, uint32_t* out_c,
                                           uint32_t rank, uint64_t* my_sync, uint64_t* const* peer_sync,
                                           uint64_t epoch, void* stream) {
  try {
    if (nsrc > 64) throw Error(GRAB_ERR_VALUE, "at most 64 shards");
    if (nq > B) throw Error(GRAB_ERR_VALUE, "owned queries exceed the block size");
    // at least one block: an owner with no queries still releases its buffer
    k_merge_topk_p2p<<<(unsigned)std::max<uint64_t>(1, div_up(nq, 128)), 128, 0, (cudaStream_t)stream>>>(
        nq, nsrc, B, k, d, id, out_d, out_i, out_c, rank, my_sync, peer_sync, epoch);
    GRAB_CHECK_LAUNCH();
    return GRAB_OK;
  } catch (const Error& e) {
    return grab_set_error(e.code, e.what());
  }
}

extern "C" GRAB_API int grab_ipc_alloc(uint64_t bytes, void** ptr, void* handle64) {
  try {
    GRAB_CUDA(cudaMalloc(ptr, bytes ? bytes : 16));
    GRAB_CUDA(cudaMemset(*ptr, 0, bytes ? bytes : 16));  // zero-filled (sync blocks start at epoch 0)
    cudaIpcMemHandle_t h;
    GRAB_CUDA(cudaIpcGetMemHandle(&h, *ptr));
    static_assert(sizeof(h) == 64, "IPC handle size");
    std::memcpy(handle64, &h, 64);
    return GRAB_OK;
  } catch (const Error& e) {
    return grab_set_error(e.code, e.what());
  }
}

extern "C" GRAB_API int grab_ipc_open(const void* handle64, void** ptr) {
  try {
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle64, 64);
    GRAB_CUDA(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
    return GRAB_OK;
  } catch (const Error& e) {
    return grab_set_error(e.code, e.what());
  }
}

extern "C" GRAB_API int grab_ipc_close(void* ptr) {
  cudaIpcCloseMemHandle(ptr);
  return GRAB_OK;
}

extern "C" GRAB_API int grab_ipc_free(void* ptr) {
  cudaFree(ptr);
  return GRAB_OK;
}

extern "C" GRAB_API int grab_shard_pack_p2p(uint64_t n, const uint32_t* qidx, const int64_t* slots,
                                            const double* dists, const int64_t* gid, uint32_t k, uint32_t rank,
                                            uint32_t world, uint32_t B, double* const* peer_d, int64_t* const* peer_i,
                                            void* stream) {
  try {
    cudaStream_t st = (cudaStream_t)stream;
    if (k == 0 || world == 0 || B == 0 || rank >= world) throw Error(GRAB_ERR_VALUE, "bad shard geometry");
    const uint64_t total = (uint64_t)world * B * k;
    k_shard_fill_p2p<<<(unsigned)div_up(total, 256), 256, 0, st>>>(total, rank, B, k, world, peer_d, peer_i);
    GRAB_CHECK_LAUNCH();
    if (n) {
      k_shard_pack_p2p<<<(unsigned)div_up(n * k, 256), 256, 0, st>>>(n, qidx, slots, dists, gid, k, rank, B, peer_d,
                                                                     peer_i);
      GRAB_CHECK_LAUNCH();
    }
    return GRAB_OK;
  } catch (const Error& e) {
    return grab_set_error(e.code, e.what());
  }
}
