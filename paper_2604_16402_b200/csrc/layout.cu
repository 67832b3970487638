// Bucket-slab layout construction, zero-shift appends, slot<->phys translation.
// Reference behaviour restated: partition map population (layout.py:143-154),
// append_batch (layout.py:181-223), load_index map rebuild (dataio.py:175-186).
#include <cstring>
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <cmath>
#include <numeric>

#include "index.cuh"

namespace grab {

size_t DevIndex::device_bytes() const {
  size_t b = n_cap * (sizeof(uint32_t) + sizeof(int32_t));
  b += phys_cap * ((size_t)dp * 4 + sizeof(Attr) + (size_t)params.k_max * 4);
  b += (size_t)m * 16 + 16;
  return b;
}

static void cfree(void* p) {
  if (p) cudaFree(p);
}

void index_alloc_slots(DevIndex& ix) {
  GRAB_CUDA(cudaMalloc(&ix.slot2phys, ix.n_cap * sizeof(uint32_t)));
  GRAB_CUDA(cudaMalloc(&ix.i2b, ix.n_cap * sizeof(int32_t)));
  GRAB_CUDA(cudaMemsetAsync(ix.slot2phys, 0xFF, ix.n_cap * sizeof(uint32_t), ix.stream));
  GRAB_CUDA(cudaMemsetAsync(ix.i2b, 0xFF, ix.n_cap * sizeof(int32_t), ix.stream));
}

static void free_phys(DevIndex& ix) {
  cfree(ix.X);
  cfree(ix.attr);
  cfree(ix.adj);
  cfree(ix.adja);
  ix.adja = nullptr;
  ix.adja_rows = 0;
  ix.adj_version++;
  ix.X = nullptr;
  ix.attr = nullptr;
  ix.adj = nullptr;
  ix.phys_cap = 0;
}

static void free_buckets(DevIndex& ix) {
  cfree(ix.bound);
  cfree(ix.bstart);
  cfree(ix.bcount);
  cfree(ix.bcum);
  ix.bound = nullptr;
  ix.bstart = ix.bcount = nullptr;
  ix.bcum = nullptr;
  ix.m_alloc = 0;
}

void index_free(DevIndex& ix) {
  free_search_ws(ix);
  free_phys(ix);
  free_buckets(ix);
  cfree(ix.slot2phys);
  cfree(ix.i2b);
  ix.slot2phys = nullptr;
  ix.i2b = nullptr;
}

// Slab capacity policy: 1/8 headroom + 32 rows, rounded to 32-row multiples so
// every slab starts 512-byte aligned (dp*4 is a multiple of 16).
static uint32_t slab_cap(uint64_t members) {
  uint64_t c = members + members / 8 + 32;
  return (uint32_t)div_up(c, 32) * 32;
}

__global__ void k_init_attr(Attr* a, uint64_t n) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i < n) {
    a[i].s = __int_as_float(0x7FC00000);  // NaN: fails every range test
    a[i].slot = kNoSlot;
  }
}

static void alloc_phys(DevIndex& ix, uint64_t rows) {
  GRAB_CUDA(cudaMalloc(&ix.X, rows * ix.dp * sizeof(float)));
  GRAB_CUDA(cudaMalloc(&ix.attr, rows * sizeof(Attr)));
  GRAB_CUDA(cudaMalloc(&ix.adj, rows * ix.params.k_max * sizeof(uint32_t)));
  GRAB_CUDA(cudaMemsetAsync(ix.X, 0, rows * ix.dp * sizeof(float), ix.stream));
  GRAB_CUDA(cudaMemsetAsync(ix.adj, 0xFF, rows * ix.params.k_max * sizeof(uint32_t), ix.stream));
  if (rows) {
    k_init_attr<<<(unsigned)div_up(rows, 256), 256, 0, ix.stream>>>(ix.attr, rows);
    GRAB_CHECK_LAUNCH();
  }
  ix.phys_cap = rows;
}

void upload_bucket_tables(DevIndex& ix) {
  uint32_t m = ix.m;
  // in place when the bucket count is unchanged (every append): stream-ordered
  // after the writer lock made ix.stream wait for in-flight readers, no
  // device-wide cudaFree / cudaMalloc synchronisation
  if (!(ix.bound && ix.bstart && ix.bcount && ix.bcum && ix.m_alloc == m)) {
    free_buckets(ix);
    GRAB_CUDA(cudaMalloc(&ix.bound, (m + 1) * sizeof(float)));
    GRAB_CUDA(cudaMalloc(&ix.bstart, std::max(m, 1u) * sizeof(uint32_t)));
    GRAB_CUDA(cudaMalloc(&ix.bcount, std::max(m, 1u) * sizeof(uint32_t)));
    GRAB_CUDA(cudaMalloc(&ix.bcum, (m + 1) * sizeof(uint64_t)));
    ix.m_alloc = m;
  }
  std::vector<uint64_t> cum(m + 1, 0);
  for (uint32_t b = 0; b < m; ++b) cum[b + 1] = cum[b] + ix.h_bcount[b];
  GRAB_CUDA(cudaMemcpyAsync(ix.bound, ix.h_bound.data(), (m + 1) * sizeof(float), cudaMemcpyHostToDevice, ix.stream));
  GRAB_CUDA(cudaMemcpyAsync(ix.bstart, ix.h_bstart.data(), m * sizeof(uint32_t), cudaMemcpyHostToDevice, ix.stream));
  GRAB_CUDA(cudaMemcpyAsync(ix.bcount, ix.h_bcount.data(), m * sizeof(uint32_t), cudaMemcpyHostToDevice, ix.stream));
  GRAB_CUDA(cudaMemcpyAsync(ix.bcum, cum.data(), (m + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice, ix.stream));
  GRAB_CUDA(cudaStreamSynchronize(ix.stream));  // `cum` is a local: the copies must have read it
}

__global__ void k_iota_u32(uint32_t* out, uint64_t n, uint32_t first) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = first + (uint32_t)i;
}

// Stable bucket sort of slots [start, start+n): returns device array of slots
// ordered by (bucket, slot), allocated on ix.stream (caller frees it there).
static uint32_t* sort_slots_by_bucket(DevIndex& ix, uint64_t start, uint64_t n) {
  cudaStream_t st = ix.stream;
  uint32_t *keys_out, *vals_in, *vals_out;
  GRAB_CUDA(cudaMallocAsync(&keys_out, std::max<uint64_t>(n, 1) * 4, st));
  GRAB_CUDA(cudaMallocAsync(&vals_in, std::max<uint64_t>(n, 1) * 4, st));
  GRAB_CUDA(cudaMallocAsync(&vals_out, std::max<uint64_t>(n, 1) * 4, st));
  if (n) {
    k_iota_u32<<<(unsigned)div_up(n, 256), 256, 0, st>>>(vals_in, n, (uint32_t)start);
    GRAB_CHECK_LAUNCH();
  }
  int bits = 1;
  while ((1u << bits) < std::max(ix.m, 2u)) ++bits;
  // bucket ids are >= 0 here: sorting their low `bits` bits as u32 keys is exact
  const uint32_t* keys_in = reinterpret_cast<const uint32_t*>(ix.i2b + start);
  size_t tmp_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys_in, keys_out, vals_in, vals_out, (int)n, 0, bits, st);
  void* tmp;
  GRAB_CUDA(cudaMallocAsync(&tmp, std::max<size_t>(tmp_bytes, 16), st));
  GRAB_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys_in, keys_out, vals_in, vals_out, (int)n, 0, bits, st));
  GRAB_CUDA(cudaFreeAsync(tmp, st));
  GRAB_CUDA(cudaFreeAsync(keys_out, st));
  GRAB_CUDA(cudaFreeAsync(vals_in, st));
  return vals_out;
}

// Place sorted slots: j-th slot of bucket b (within this batch) goes to
// phys = bstart[b] + base[b] + (j - first[b]).
__global__ void k_place(const uint32_t* sorted, uint64_t n, const int32_t* i2b, const uint32_t* bstart,
                        const uint32_t* base, const uint64_t* first, uint32_t* slot2phys, Attr* attr,
                        float* X, uint32_t dp, const float* Xsrc, const float* Ssrc, uint32_t dim,
                        uint64_t src_slot0) {
  uint64_t j = blockIdx.x;
  if (j >= n) return;
  uint32_t slot = sorted[j];
  int32_t b = i2b[slot];
  uint32_t phys = bstart[b] + base[b] + (uint32_t)(j - first[b]);
  const float* src = Xsrc + (uint64_t)(slot - src_slot0) * dim;
  float* dst = X + (uint64_t)phys * dp;
  for (uint32_t c = threadIdx.x; c < dp; c += blockDim.x) dst[c] = c < dim ? src[c] : 0.f;
  if (threadIdx.x == 0) {
    slot2phys[slot] = phys;
    attr[phys].s = Ssrc[slot - src_slot0];
    attr[phys].slot = slot;
  }
}

// per_bucket: the batch's row count per bucket (from the caller's bucket ids)
static void place_batch(DevIndex& ix, const float* Xsrc, const float* Ssrc, uint64_t start, uint64_t n,
                        const std::vector<uint32_t>& base, const std::vector<uint32_t>& per_bucket) {
  cudaStream_t st = ix.stream;
  uint32_t* sorted = sort_slots_by_bucket(ix, start, n);
  // first position of each bucket in the sorted batch
  std::vector<uint64_t> first(ix.m + 1, 0);
  for (uint32_t b = 0; b < ix.m; ++b) first[b + 1] = first[b] + per_bucket[b];
  // one small table upload: base [m] u32 | bstart [m] u32 | first [m+1] u64
  const size_t tb = (size_t)ix.m * 8 + (size_t)(ix.m + 1) * 8;
  std::vector<uint8_t> host(tb);
  std::memcpy(host.data(), base.data(), ix.m * 4);
  std::memcpy(host.data() + ix.m * 4, ix.h_bstart.data(), ix.m * 4);
  std::memcpy(host.data() + ix.m * 8, first.data(), (ix.m + 1) * 8);
  uint8_t* d;
  GRAB_CUDA(cudaMallocAsync(&d, tb, st));
  GRAB_CUDA(cudaMemcpyAsync(d, host.data(), tb, cudaMemcpyHostToDevice, st));
  if (n) {
    k_place<<<(unsigned)n, 32, 0, st>>>(sorted, n, ix.i2b, (const uint32_t*)(d + ix.m * 4), (const uint32_t*)d,
                                        (const uint64_t*)(d + ix.m * 8), ix.slot2phys, ix.attr, ix.X, ix.dp, Xsrc,
                                        Ssrc, ix.dim, start);
    GRAB_CHECK_LAUNCH();
  }
  GRAB_CUDA(cudaFreeAsync(sorted, st));
  GRAB_CUDA(cudaFreeAsync(d, st));
  GRAB_CUDA(cudaStreamSynchronize(st));  // `host` is a local: the copy must have read it
}

void layout_from_slots(DevIndex& ix, const float* X_slot, const float* S_slot, uint64_t count,
                       const std::vector<uint32_t>& sizes) {
  free_phys(ix);
  ix.m = (uint32_t)sizes.size();
  ix.h_bcount = sizes;
  ix.h_bcap.resize(ix.m);
  ix.h_bstart.resize(ix.m);
  uint64_t total = 0;
  for (uint32_t b = 0; b < ix.m; ++b) {
    ix.h_bstart[b] = (uint32_t)total;
    ix.h_bcap[b] = slab_cap(sizes[b]);
    total += ix.h_bcap[b];
  }
  if (total >= 0xFFFFFFFFull) throw Error(GRAB_ERR_CAPACITY, "physical rows exceed u32 id space");
  alloc_phys(ix, total);
  std::vector<uint32_t> base(ix.m, 0);
  place_batch(ix, X_slot, S_slot, 0, count, base, sizes);
  ix.count = count;
  upload_bucket_tables(ix);
}

// Move every slab to a new allocation with fresh headroom (after which the
// pending batch `extra[b]` fits), remapping adjacency phys ids.
__global__ void k_move_rows(const float* X0, const Attr* A0, const uint32_t* adj0, uint64_t rows0,
                            const uint32_t* remap, float* X1, Attr* A1, uint32_t* adj1, uint32_t dp,
                            uint32_t k_max, uint32_t* slot2phys) {
  uint64_t p = blockIdx.x;
  if (p >= rows0) return;
  uint32_t q = remap[p];
  if (q == kSentinel) return;
  for (uint32_t c = threadIdx.x; c < dp; c += blockDim.x) X1[(uint64_t)q * dp + c] = X0[p * dp + c];
  for (uint32_t j = threadIdx.x; j < k_max; j += blockDim.x) {
    uint32_t v = adj0[p * k_max + j];
    adj1[(uint64_t)q * k_max + j] = v == kSentinel ? kSentinel : remap[v];
  }
  if (threadIdx.x == 0) {
    A1[q] = A0[p];
    slot2phys[A0[p].slot] = q;
  }
}

__global__ void k_build_remap(const Attr* A0, uint64_t rows0, const uint32_t* phys_bucket_of,
                              const uint32_t* old_start, const uint32_t* new_start, uint32_t* remap) {
  uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (p >= rows0) return;
  if (A0[p].slot == kNoSlot) {
    remap[p] = kSentinel;
    return;
  }
  uint32_t b = phys_bucket_of[p];
  remap[p] = new_start[b] + (uint32_t)(p - old_start[b]);
}

__global__ void k_phys_bucket(const uint32_t* starts, const uint32_t* caps, uint32_t m, uint32_t* out) {
  uint32_t b = blockIdx.x;
  if (b >= m) return;
  for (uint32_t i = threadIdx.x; i < caps[b]; i += blockDim.x) out[starts[b] + i] = b;
}

static void relayout(DevIndex& ix, const std::vector<uint32_t>& extra) {
  uint32_t m = ix.m;
  std::vector<uint32_t> nstart(m), ncap(m);
  uint64_t total = 0;
  for (uint32_t b = 0; b < m; ++b) {
    nstart[b] = (uint32_t)total;
    uint64_t want = (uint64_t)ix.h_bcount[b] + extra[b];
    // geometric growth: a relayout leaves 50 % headroom so append-only batches
    // relayout O(log) times, not once per batch
    ncap[b] = std::max(ix.h_bcap[b], slab_cap(want + want / 2));
    total += ncap[b];
  }
  if (total >= 0xFFFFFFFFull) throw Error(GRAB_ERR_CAPACITY, "physical rows exceed u32 id space");
  uint64_t rows0 = ix.phys_cap;
  float* X0 = ix.X;
  Attr* A0 = ix.attr;
  uint32_t* adj0 = ix.adj;
  ix.X = nullptr;
  ix.attr = nullptr;
  ix.adj = nullptr;
  ix.adj_version++;
  alloc_phys(ix, total);
  uint32_t *d_os, *d_ns, *d_oc, *d_pb, *d_remap;
  GRAB_CUDA(cudaMalloc(&d_os, m * 4));
  GRAB_CUDA(cudaMalloc(&d_ns, m * 4));
  GRAB_CUDA(cudaMalloc(&d_oc, m * 4));
  GRAB_CUDA(cudaMalloc(&d_pb, std::max<uint64_t>(rows0, 1) * 4));
  GRAB_CUDA(cudaMalloc(&d_remap, std::max<uint64_t>(rows0, 1) * 4));
  GRAB_CUDA(cudaMemcpyAsync(d_os, ix.h_bstart.data(), m * 4, cudaMemcpyHostToDevice, ix.stream));
  GRAB_CUDA(cudaMemcpyAsync(d_ns, nstart.data(), m * 4, cudaMemcpyHostToDevice, ix.stream));
  GRAB_CUDA(cudaMemcpyAsync(d_oc, ix.h_bcap.data(), m * 4, cudaMemcpyHostToDevice, ix.stream));
  k_phys_bucket<<<m, 256, 0, ix.stream>>>(d_os, d_oc, m, d_pb);
  GRAB_CHECK_LAUNCH();
  if (rows0) {
    k_build_remap<<<(unsigned)div_up(rows0, 256), 256, 0, ix.stream>>>(A0, rows0, d_pb, d_os, d_ns, d_remap);
    GRAB_CHECK_LAUNCH();
    k_move_rows<<<(unsigned)rows0, 128, 0, ix.stream>>>(X0, A0, adj0, rows0, d_remap, ix.X, ix.attr, ix.adj,
                                                         ix.dp, ix.params.k_max, ix.slot2phys);
    GRAB_CHECK_LAUNCH();
  }
  GRAB_CUDA(cudaStreamSynchronize(ix.stream));
  cudaFree(d_os);
  cudaFree(d_ns);
  cudaFree(d_oc);
  cudaFree(d_pb);
  cudaFree(d_remap);
  cudaFree(X0);
  cudaFree(A0);
  cudaFree(adj0);
  ix.h_bstart = nstart;
  ix.h_bcap = ncap;
}

void layout_append(DevIndex& ix, const float* X_new, const float* S_new, uint64_t start, uint64_t b) {
  std::vector<int32_t> hb(b);
  // the bucket ids were computed on ix.stream (non-blocking): read them on that
  // stream -- a legacy-stream cudaMemcpy does not wait for it and could see the
  // -1 fill, indexing `extra` out of bounds
  GRAB_CUDA(cudaMemcpyAsync(hb.data(), ix.i2b + start, b * 4, cudaMemcpyDeviceToHost, ix.stream));
  GRAB_CUDA(cudaStreamSynchronize(ix.stream));
  std::vector<uint32_t> extra(ix.m, 0);
  for (uint64_t i = 0; i < b; ++i) {
    if (hb[i] < 0 || (uint32_t)hb[i] >= ix.m) throw Error(GRAB_ERR_CUDA, "append: bucket id out of range");
    extra[hb[i]]++;
  }
  bool overflow = false;
  for (uint32_t k = 0; k < ix.m; ++k)
    if ((uint64_t)ix.h_bcount[k] + extra[k] > ix.h_bcap[k]) overflow = true;
  if (overflow) relayout(ix, extra);
  std::vector<uint32_t> base = ix.h_bcount;
  place_batch(ix, X_new, S_new, start, b, base, extra);
  for (uint32_t k = 0; k < ix.m; ++k) ix.h_bcount[k] += extra[k];
  ix.count = start + b;
  upload_bucket_tables(ix);
}

__global__ void k_adj_to_phys(const uint32_t* adj_slot, uint64_t n, uint32_t k_max, const uint32_t* s2p,
                              uint32_t* adj) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= n * k_max) return;
  uint64_t u = i / k_max, j = i % k_max;
  uint32_t v = adj_slot[i];
  adj[(uint64_t)s2p[u] * k_max + j] = (v == kSentinel || v >= n) ? kSentinel : s2p[v];
}

void adjacency_slot_to_phys(DevIndex& ix, const uint32_t* adj_slot_dev, uint64_t n) {
  uint64_t tot = n * ix.params.k_max;
  if (!tot) return;
  k_adj_to_phys<<<(unsigned)div_up(tot, 256), 256, 0, ix.stream>>>(adj_slot_dev, n, ix.params.k_max,
                                                                   ix.slot2phys, ix.adj);
  GRAB_CHECK_LAUNCH();
}

__global__ void k_adj_to_slot(const uint32_t* adj, const Attr* attr, const uint32_t* s2p, uint64_t start,
                              uint64_t n, uint32_t k_max, uint32_t* out) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= n * k_max) return;
  uint64_t u = start + i / k_max, j = i % k_max;
  uint32_t v = adj[(uint64_t)s2p[u] * k_max + j];
  out[i] = v == kSentinel ? kSentinel : attr[v].slot;
}

void adjacency_phys_to_slot(const DevIndex& ix, uint32_t* out, uint64_t start, uint64_t n) {
  uint64_t tot = n * ix.params.k_max;
  if (!tot) return;
  k_adj_to_slot<<<(unsigned)div_up(tot, 256), 256, 0, ix.stream>>>(ix.adj, ix.attr, ix.slot2phys, start, n,
                                                                    ix.params.k_max, out);
  GRAB_CHECK_LAUNCH();
}

__global__ void k_gather_rows(const float* X, const Attr* attr, const uint32_t* s2p, uint64_t start,
                              uint64_t n, uint32_t dim, uint32_t dp, float* Xo, float* So) {
  uint64_t u = blockIdx.x;
  if (u >= n) return;
  uint32_t p = s2p[start + u];
  if (Xo)
    for (uint32_t c = threadIdx.x; c < dim; c += blockDim.x) Xo[u * dim + c] = X[(uint64_t)p * dp + c];
  if (So && threadIdx.x == 0) So[u] = attr[p].s;
}

void gather_slot_rows(const DevIndex& ix, float* Xo, float* So, uint64_t start, uint64_t n) {
  if (!n) return;
  k_gather_rows<<<(unsigned)n, 128, 0, ix.stream>>>(ix.X, ix.attr, ix.slot2phys, start, n, ix.dim, ix.dp, Xo, So);
  GRAB_CHECK_LAUNCH();
}

}  // namespace grab
