// extern "C" boundary (include/grab.h). Converts exceptions to GRAB_ERR_*
// codes, stages host buffers, and dispatches to the kernels.
#include <algorithm>
#include <chrono>
#include <cstring>
#include <memory>
#include <map>
#include <mutex>
#include <shared_mutex>
#include <string>
#include <vector>

#include "index.cuh"
#include "ops.cuh"
#include "rng.cuh"
#include "search.cuh"

using namespace grab;

// Concurrency (layout.py:238-239): search / brute force / reads are
// concurrent readers, build / import / insert / append exclusive topology
// writers. Readers hold `rw` shared while they enqueue and record `done` on
// their stream; a writer takes `rw` exclusive and makes its own stream wait for
// every reader stream's last event before it rewires rows or relayouts (frees)
// buffers, so no in-flight search ever reads a freed or half-rewired array.
// Writers synchronize their stream before returning, so readers that start
// afterwards see the last published count and the new pointers.
struct grab_index {
  DevIndex ix;
  std::shared_mutex rw;
  std::mutex readers_mu;
  std::map<cudaStream_t, cudaEvent_t> readers;  // reader stream -> its last enqueued work
  ~grab_index() {
    for (auto& kv : readers) cudaEventDestroy(kv.second);
  }
};

namespace {
struct ReadLock {
  grab_index* h;
  std::shared_lock<std::shared_mutex> lk;
  explicit ReadLock(const grab_index* hc) : h(const_cast<grab_index*>(hc)), lk(h->rw) {}
  // after enqueueing on `st`: remember it so a later writer can wait for it
  void done(cudaStream_t st) {
    std::lock_guard<std::mutex> g(h->readers_mu);
    cudaEvent_t& ev = h->readers[st];
    if (!ev) GRAB_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    GRAB_CUDA(cudaEventRecord(ev, st));
  }
};
struct WriteLock {
  std::unique_lock<std::shared_mutex> lk;
  explicit WriteLock(grab_index* h) : lk(h->rw) {
    std::lock_guard<std::mutex> g(h->readers_mu);
    for (auto& kv : h->readers) GRAB_CUDA(cudaStreamWaitEvent(h->ix.stream, kv.second, 0));
  }
};
}  // namespace

static thread_local std::string g_err;

extern "C" const char* grab_last_error(void) { return g_err.c_str(); }

namespace grab {
// for entry points defined in other translation units (shard.cu)
int grab_set_error(int code, const char* msg) {
  g_err = msg;
  return code;
}
}  // namespace grab

template <class F>
static int guarded(F&& f) {
  try {
    f();
    return GRAB_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return GRAB_ERR_CUDA;
  }
}

// RAII device scratch
struct DBuf {
  void* p = nullptr;
  cudaStream_t st = nullptr;
  DBuf() = default;
  DBuf(size_t bytes, cudaStream_t s) : st(s) {
    if (bytes) GRAB_CUDA(cudaMallocAsync(&p, bytes, s));
  }
  ~DBuf() {
    if (p) cudaFreeAsync(p, st);
  }
  template <class T>
  T* as() const {
    return (T*)p;
  }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
};

static void set_device(const DevIndex& ix) { GRAB_CUDA(cudaSetDevice(ix.device)); }

static void check_handle(const grab_index* h) {
  if (!h) throw Error(GRAB_ERR_VALUE, "null index handle");
}

static void check_build_params(const grab_build_params* p) {
  if (!p) throw Error(GRAB_ERR_VALUE, "null build params");
  if (!(p->k_local > 0 && p->k_local <= p->k_max))
    throw Error(GRAB_ERR_VALUE, "need 0 < k_local <= k_max, got " + std::to_string(p->k_local) + "/" +
                                    std::to_string(p->k_max));
  if (p->bucket_capacity < 1) throw Error(GRAB_ERR_VALUE, "bucket_capacity must be >= 1");
  if (!(p->proximal_fraction >= 0.0 && p->proximal_fraction <= 1.0))
    throw Error(GRAB_ERR_VALUE, "proximal_fraction must lie in [0, 1]");
  if (!(p->proximal_window > 0.0 && p->proximal_window <= 1.0))
    throw Error(GRAB_ERR_VALUE, "proximal_window must lie in (0, 1]");
  if (!(p->alpha > 0.0 && p->alpha <= 1.0)) throw Error(GRAB_ERR_VALUE, "alpha must lie in (0, 1]");
}

extern "C" int grab_create(int device, uint32_t dim, uint64_t capacity, const grab_build_params* params,
                           grab_index** out) {
  return guarded([&] {
    if (!out) throw Error(GRAB_ERR_VALUE, "null out");
    if (capacity < 1 || dim < 1) throw Error(GRAB_ERR_VALUE, "capacity and dim must be >= 1");
    if (capacity >= 0xFFFFFFFFull) throw Error(GRAB_ERR_VALUE, "capacity exceeds u32 slot space");
    check_build_params(params);
    auto h = std::make_unique<grab_index>();
    DevIndex& ix = h->ix;
    ix.device = device;
    GRAB_CUDA(cudaSetDevice(device));
    GRAB_CUDA(cudaDeviceGetAttribute(&ix.num_sms, cudaDevAttrMultiProcessorCount, device));
    GRAB_CUDA(cudaStreamCreateWithFlags(&ix.stream, cudaStreamNonBlocking));
    {
      // keep stream-ordered scratch (visited tables, staging) mapped across calls
      cudaMemPool_t pool;
      GRAB_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
      uint64_t keep = ~0ull;
      GRAB_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    }
    ix.dim = dim;
    ix.dp = (dim + 3) / 4 * 4;
    ix.n_cap = capacity;
    ix.params = *params;
    ix.ids.assign(capacity, -1);
    index_alloc_slots(ix);
    upload_pcg_jump_tables();
    GRAB_CUDA(cudaStreamSynchronize(ix.stream));
    *out = h.release();
  });
}

extern "C" void grab_destroy(grab_index* h) {
  if (!h) return;
  cudaSetDevice(h->ix.device);
  cudaStreamSynchronize(h->ix.stream);
  index_free(h->ix);
  cudaStreamDestroy(h->ix.stream);
  delete h;
}

extern "C" int grab_get_info(const grab_index* h, grab_info_t* out) {
  return guarded([&] {
    check_handle(h);
    const DevIndex& ix = h->ix;
    std::memset(out, 0, sizeof(*out));
    out->count = ix.count;
    out->capacity = ix.n_cap;
    out->dim = ix.dim;
    out->k_max = ix.params.k_max;
    out->k_local = ix.params.k_local;
    out->m = ix.m;
    out->built = ix.built ? 1 : 0;
    out->phys_capacity = ix.phys_cap;
    out->device_bytes = ix.device_bytes();
  });
}

extern "C" int grab_sync(grab_index* h) {
  return guarded([&] {
    check_handle(h);
    set_device(h->ix);
    GRAB_CUDA(cudaStreamSynchronize(h->ix.stream));
  });
}

// Copy (or alias) rows of `dim` floats into a dp-padded device buffer.
static const float* padded_rows(const DevIndex& ix, const float* src, uint64_t n, uint32_t mem, DBuf& keep,
                                cudaStream_t st) {
  if (mem == GRAB_MEM_DEVICE && ix.dp == ix.dim) return src;
  keep.~DBuf();
  new (&keep) DBuf(std::max<uint64_t>(n, 1) * ix.dp * 4, st);
  float* dst = keep.as<float>();
  if (ix.dp == ix.dim) {
    GRAB_CUDA(cudaMemcpyAsync(dst, src, n * ix.dim * 4, cudaMemcpyHostToDevice, st));
  } else {
    GRAB_CUDA(cudaMemsetAsync(dst, 0, n * ix.dp * 4, st));
    GRAB_CUDA(cudaMemcpy2DAsync(dst, ix.dp * 4, src, ix.dim * 4, ix.dim * 4, n,
                                mem == GRAB_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
  }
  return dst;
}

template <class T>
static const T* stage_in(const T* src, uint64_t n, uint32_t mem, DBuf& keep, cudaStream_t st) {
  if (!src || mem == GRAB_MEM_DEVICE) return src;
  keep.~DBuf();
  new (&keep) DBuf(std::max<uint64_t>(n, 1) * sizeof(T), st);
  GRAB_CUDA(cudaMemcpyAsync(keep.p, src, n * sizeof(T), cudaMemcpyHostToDevice, st));
  return keep.as<T>();
}

template <class T>
static T* stage_out(T* dst, uint64_t n, uint32_t mem, DBuf& keep, cudaStream_t st) {
  if (!dst || mem == GRAB_MEM_DEVICE) return dst;
  keep.~DBuf();
  new (&keep) DBuf(std::max<uint64_t>(n, 1) * sizeof(T), st);
  return keep.as<T>();
}

template <class T>
static void copy_back(T* host, const DBuf& b, uint64_t n, uint32_t mem, cudaStream_t st) {
  if (!host || mem == GRAB_MEM_DEVICE) return;
  GRAB_CUDA(cudaMemcpyAsync(host, b.p, n * sizeof(T), cudaMemcpyDeviceToHost, st));
}

// Device address of a page-locked host buffer (cudaHostAlloc / cudaHostRegister,
// e.g. torch pin_memory), else nullptr. Null pointers count as mapped.
static const void* mapped_host(const void* p) {
  if (!p) return nullptr;
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return at.type == cudaMemoryTypeHost ? at.devicePointer : nullptr;
}

static uint64_t live_of(const DevIndex& ix, uint64_t live_count) {
  return live_count == GRAB_LIVE_ALL ? ix.count : std::min<uint64_t>(live_count, ix.count);
}

extern "C" int grab_search(const grab_index* h, const float* queries, uint64_t nq, const double* lower,
                           const double* upper, uint64_t range_stride, const grab_search_params* p,
                           const uint64_t* seeds, uint64_t seed_base, uint64_t ordinal0, uint64_t live_count,
                           int64_t* out_slots, double* out_dists, uint32_t* out_counts,
                           grab_search_stats* out_stats, uint32_t mem, void* stream) {
  return guarded([&] {
    check_handle(h);
    ReadLock rl(h);
    const DevIndex& ix = h->ix;
    set_device(ix);
    if (!p) throw Error(GRAB_ERR_VALUE, "null search params");
    if (p->k < 1 || p->k > p->itopk)
      throw Error(GRAB_ERR_VALUE, "need 1 <= k <= itopk, got k=" + std::to_string(p->k) + " itopk=" +
                                      std::to_string(p->itopk));
    if (p->search_width < 1) throw Error(GRAB_ERR_VALUE, "search_width must be >= 1");
    if (p->itopk > 2048) throw Error(GRAB_ERR_VALUE, "itopk > 2048 not supported");
    if (nq == 0) return;
    if (nq >= 0xFFFFFFFFull) throw Error(GRAB_ERR_VALUE, "too many queries in one batch");
    cudaStream_t st = mem == GRAB_MEM_DEVICE ? (cudaStream_t)stream : ix.stream;  // device mode: the caller's stream (NULL = legacy default)
    uint64_t nr = range_stride ? nq : 1;
    if (mem == GRAB_MEM_HOST) {
      for (uint64_t i = 0; i < nr; ++i)
        if (!(lower[i * range_stride] <= upper[i * range_stride]))
          throw Error(GRAB_ERR_VALUE, "invalid range: lower > upper");
    }
    // Zero-copy when every host buffer is page-locked: the kernel reads each
    // query row / bound over the host link when its warp starts the query and
    // stores the results straight into host memory, so the copies overlap the
    // search instead of bracketing it (GRAB_NO_ZERO_COPY=1 disables).
    bool zc = mem == GRAB_MEM_HOST && ix.dp == ix.dim && !getenv("GRAB_NO_ZERO_COPY");
    const void* zq = nullptr;
    const void *zlo = nullptr, *zhi = nullptr, *zsd = nullptr, *zs = nullptr, *zd = nullptr, *zc_ = nullptr,
               *zst = nullptr;
    if (zc) {
      zq = mapped_host(queries);
      zlo = mapped_host(lower);
      zhi = mapped_host(upper);
      zsd = mapped_host(seeds);
      zs = mapped_host(out_slots);
      zd = mapped_host(out_dists);
      zc_ = mapped_host(out_counts);
      zst = mapped_host(out_stats);
      zc = zq && ((uintptr_t)zq & 15) == 0 && zlo && zhi && (!seeds || zsd) && zs && zd && zc_ && (!out_stats || zst);
    }
    DBuf bq, blo, bhi, bseed, bs, bd, bc, bst;
    SearchArgs a{};
    a.X = ix.X;
    a.attr = ix.attr;
    a.adj = ix.adj;
    a.dp = ix.dp;
    a.k_max = ix.params.k_max;
    a.bound = ix.bound;
    a.m = ix.built ? ix.m : 0;
    a.bstart = ix.bstart;
    a.bcount = ix.bcount;
    a.bcum = ix.bcum;
    a.n_live = live_of(ix, live_count);
    const uint32_t smem = zc ? (uint32_t)GRAB_MEM_DEVICE : mem;  // staging mode of the buffers
    a.Q = zc ? (const float*)zq : padded_rows(ix, queries, nq, mem, bq, st);
    a.lower = stage_in(zc ? (const double*)zlo : lower, (nr - 1) * range_stride + 1, smem, blo, st);
    a.upper = stage_in(zc ? (const double*)zhi : upper, (nr - 1) * range_stride + 1, smem, bhi, st);
    a.range_stride = range_stride;
    a.seeds = stage_in(zc ? (const uint64_t*)zsd : seeds, nq, smem, bseed, st);
    a.seed_base = seed_base;
    a.ordinal0 = ordinal0;
    a.k = p->k;
    a.itopk = p->itopk;
    a.width = p->search_width;
    a.max_iter = p->max_iterations;
    a.want = p->seed_count ? p->seed_count : std::min<uint32_t>(p->itopk, 32);
    a.nwork = (uint32_t)nq;
    a.out_slots = stage_out(zc ? (int64_t*)zs : out_slots, nq * p->k, smem, bs, st);
    a.out_dists = stage_out(zc ? (double*)zd : out_dists, nq * p->k, smem, bd, st);
    a.out_counts = stage_out(zc ? (uint32_t*)zc_ : out_counts, nq, smem, bc, st);
    a.out_stats = stage_out(zc ? (grab_search_stats*)zst : out_stats, nq, smem, bst, st);
    run_search(ix, a, st);
    copy_back(out_slots, bs, nq * p->k, smem, st);
    copy_back(out_dists, bd, nq * p->k, smem, st);
    copy_back(out_counts, bc, nq, smem, st);
    copy_back(out_stats, bst, nq, smem, st);
    rl.done(st);
    if (mem == GRAB_MEM_HOST) GRAB_CUDA(cudaStreamSynchronize(st));
  });
}

extern "C" int grab_brute_force(const grab_index* h, const float* queries, uint64_t nq, const double* lower,
                                const double* upper, uint64_t range_stride, uint32_t k, uint64_t live_count,
                                int64_t* out_slots, double* out_dists, uint32_t* out_counts, uint32_t mem,
                                void* stream) {
  return guarded([&] {
    check_handle(h);
    ReadLock rl(h);
    const DevIndex& ix = h->ix;
    set_device(ix);
    if (k < 1) throw Error(GRAB_ERR_VALUE, "k must be >= 1");
    if (nq == 0) return;
    cudaStream_t st = mem == GRAB_MEM_DEVICE ? (cudaStream_t)stream : ix.stream;  // device mode: the caller's stream (NULL = legacy default)
    uint64_t nr = range_stride ? nq : 1;
    DBuf bq, blo, bhi, bs, bd, bc;
    const float* Q = padded_rows(ix, queries, nq, mem, bq, st);
    const double* lo = stage_in(lower, (nr - 1) * range_stride + 1, mem, blo, st);
    const double* hi = stage_in(upper, (nr - 1) * range_stride + 1, mem, bhi, st);
    int64_t* os = stage_out(out_slots, nq * k, mem, bs, st);
    double* od = stage_out(out_dists, nq * k, mem, bd, st);
    uint32_t* oc = stage_out(out_counts, nq, mem, bc, st);
    DevIndex view = ix;  // shallow: m = 0 when never built
    if (!ix.built) view.m = 0;
    run_bruteforce(view, Q, nq, lo, hi, range_stride, k, live_of(ix, live_count), os, od, oc, st);
    copy_back(out_slots, bs, nq * k, mem, st);
    copy_back(out_dists, bd, nq * k, mem, st);
    copy_back(out_counts, bc, nq, mem, st);
    rl.done(st);
    if (mem == GRAB_MEM_HOST) GRAB_CUDA(cudaStreamSynchronize(st));
    // `view` shares pointers with ix; release them without freeing
    view.X = nullptr;
  });
}

extern "C" int grab_bucket_select(const grab_index* h, const double* lower, const double* upper, uint64_t n,
                                  int32_t* out_lo, int32_t* out_hi, uint32_t mem, void* stream) {
  return guarded([&] {
    check_handle(h);
    ReadLock rl(h);
    const DevIndex& ix = h->ix;
    set_device(ix);
    if (!ix.built) throw Error(GRAB_ERR_STATE, "index has no bucket metadata (never built)");
    if (!n) return;
    cudaStream_t st = mem == GRAB_MEM_DEVICE ? (cudaStream_t)stream : ix.stream;  // device mode: the caller's stream (NULL = legacy default)
    DBuf a, b, c, d;
    const double* lo = stage_in(lower, n, mem, a, st);
    const double* hi = stage_in(upper, n, mem, b, st);
    int32_t* ol = stage_out(out_lo, n, mem, c, st);
    int32_t* oh = stage_out(out_hi, n, mem, d, st);
    launch_bucket_select(ix, lo, hi, n, ol, oh, st);
    copy_back(out_lo, c, n, mem, st);
    copy_back(out_hi, d, n, mem, st);
    rl.done(st);
    if (mem == GRAB_MEM_HOST) GRAB_CUDA(cudaStreamSynchronize(st));
  });
}

extern "C" int grab_bucket_ids(const grab_index* h, const float* scalars, uint64_t n, int32_t* out, uint32_t mem,
                               void* stream) {
  return guarded([&] {
    check_handle(h);
    ReadLock rl(h);
    const DevIndex& ix = h->ix;
    set_device(ix);
    if (!ix.built) throw Error(GRAB_ERR_STATE, "index has no bucket metadata (never built)");
    if (!n) return;
    cudaStream_t st = mem == GRAB_MEM_DEVICE ? (cudaStream_t)stream : ix.stream;  // device mode: the caller's stream (NULL = legacy default)
    DBuf a, c;
    const float* s = stage_in(scalars, n, mem, a, st);
    int32_t* o = stage_out(out, n, mem, c, st);
    launch_bucket_ids(ix, s, n, o, st);
    copy_back(out, c, n, mem, st);
    rl.done(st);
    if (mem == GRAB_MEM_HOST) GRAB_CUDA(cudaStreamSynchronize(st));
  });
}

extern "C" int grab_partition(int device, const float* scalars, uint64_t n, uint32_t target_capacity, int strategy,
                              float* out_boundaries, uint32_t max_boundaries, uint32_t* out_m, int32_t* out_ids,
                              uint32_t mem, void* stream) {
  return guarded([&] {
    if (!out_boundaries || !out_m) throw Error(GRAB_ERR_VALUE, "null output");
    GRAB_CUDA(cudaSetDevice(device));
    cudaStream_t st = mem == GRAB_MEM_DEVICE ? (cudaStream_t)stream : (cudaStream_t)0;
    DBuf a, c;
    const float* s = stage_in(scalars, n, mem, a, st);
    const std::vector<float> edges = partition_edges_device(s, n, target_capacity, strategy, st);
    if (edges.size() > max_boundaries) throw Error(GRAB_ERR_VALUE, "boundary buffer too small");
    std::copy(edges.begin(), edges.end(), out_boundaries);
    *out_m = (uint32_t)edges.size() - 1;
    if (out_ids && n) {
      DBuf db(edges.size() * 4, st);
      GRAB_CUDA(cudaMemcpyAsync(db.p, edges.data(), edges.size() * 4, cudaMemcpyHostToDevice, st));
      DevIndex tmp;
      tmp.bound = db.as<float>();
      tmp.m = *out_m;
      int32_t* o = stage_out(out_ids, n, mem, c, st);
      launch_bucket_ids(tmp, s, n, o, st);
      copy_back(out_ids, c, n, mem, st);
      GRAB_CUDA(cudaStreamSynchronize(st));
    }
  });
}

extern "C" int grab_import(grab_index* h, uint64_t n, const float* X, const float* scalars,
                           const uint32_t* adjacency, const float* boundaries, uint32_t m, const int32_t* i2b,
                           const uint32_t* b2i_flat, const uint64_t* b2i_offsets) {
  return guarded([&] {
    check_handle(h);
    WriteLock lk(h);
    DevIndex& ix = h->ix;
    set_device(ix);
    if (n > ix.n_cap) throw Error(GRAB_ERR_CAPACITY, "import exceeds capacity");
    if (m < 1) throw Error(GRAB_ERR_VALUE, "need at least one bucket");
    // M_B2I must list every slot once, ascending within a bucket (the order
    // partition/append produce); the device layout relies on it.
    std::vector<uint32_t> sizes(m);
    std::vector<uint8_t> seen(n, 0);
    for (uint32_t b = 0; b < m; ++b) {
      sizes[b] = (uint32_t)(b2i_offsets[b + 1] - b2i_offsets[b]);
      for (uint64_t j = b2i_offsets[b]; j < b2i_offsets[b + 1]; ++j) {
        uint32_t s = b2i_flat[j];
        if (s >= n || seen[s] || i2b[s] != (int32_t)b)
          throw Error(GRAB_ERR_VALUE, "bucket membership inconsistent with index_to_bucket");
        if (j > b2i_offsets[b] && b2i_flat[j - 1] >= s)
          throw Error(GRAB_ERR_VALUE, "bucket member lists must be in ascending slot order");
        seen[s] = 1;
      }
    }
    if (b2i_offsets[m] != n) throw Error(GRAB_ERR_VALUE, "bucket lists do not cover the live slots");
    cudaStream_t st = ix.stream;
    ix.m = m;
    ix.h_bound.assign(boundaries, boundaries + m + 1);
    GRAB_CUDA(cudaMemsetAsync(ix.i2b, 0xFF, ix.n_cap * 4, st));
    GRAB_CUDA(cudaMemcpyAsync(ix.i2b, i2b, n * 4, cudaMemcpyHostToDevice, st));
    DBuf dx(std::max<uint64_t>(n, 1) * ix.dim * 4, st), ds(std::max<uint64_t>(n, 1) * 4, st),
        da(std::max<uint64_t>(n, 1) * ix.params.k_max * 4, st);
    GRAB_CUDA(cudaMemcpyAsync(dx.p, X, n * ix.dim * 4, cudaMemcpyHostToDevice, st));
    GRAB_CUDA(cudaMemcpyAsync(ds.p, scalars, n * 4, cudaMemcpyHostToDevice, st));
    GRAB_CUDA(cudaMemcpyAsync(da.p, adjacency, n * ix.params.k_max * 4, cudaMemcpyHostToDevice, st));
    layout_from_slots(ix, dx.as<float>(), ds.as<float>(), n, sizes);
    adjacency_slot_to_phys(ix, da.as<uint32_t>(), n);
    for (uint64_t i = 0; i < n; ++i) ix.ids[i] = (int64_t)i;
    ix.count = n;
    ix.built = true;
    ix.adj_version++;
    GRAB_CUDA(cudaStreamSynchronize(st));
  });
}

extern "C" int grab_read(const grab_index* h, int what, uint64_t start, uint64_t count, void* out) {
  return guarded([&] {
    check_handle(h);
    ReadLock rl(h);
    const DevIndex& ix = h->ix;
    set_device(ix);
    cudaStream_t st = ix.stream;
    switch (what) {
      case GRAB_ARR_X:
      case GRAB_ARR_SCALARS: {
        if (start + count > ix.count) throw Error(GRAB_ERR_VALUE, "read past count");
        size_t el = what == GRAB_ARR_X ? ix.dim : 1;
        DBuf b(std::max<uint64_t>(count, 1) * el * 4, st);
        if (what == GRAB_ARR_X)
          gather_slot_rows(ix, b.as<float>(), nullptr, start, count);
        else
          gather_slot_rows(ix, nullptr, b.as<float>(), start, count);
        GRAB_CUDA(cudaMemcpyAsync(out, b.p, count * el * 4, cudaMemcpyDeviceToHost, st));
        break;
      }
      case GRAB_ARR_ADJ: {
        if (start + count > ix.count) throw Error(GRAB_ERR_VALUE, "read past count");
        DBuf b(std::max<uint64_t>(count, 1) * ix.params.k_max * 4, st);
        adjacency_phys_to_slot(ix, b.as<uint32_t>(), start, count);
        GRAB_CUDA(cudaMemcpyAsync(out, b.p, count * ix.params.k_max * 4, cudaMemcpyDeviceToHost, st));
        break;
      }
      case GRAB_ARR_I2B:
        if (start + count > ix.n_cap) throw Error(GRAB_ERR_VALUE, "read past capacity");
        GRAB_CUDA(cudaMemcpyAsync(out, ix.i2b + start, count * 4, cudaMemcpyDeviceToHost, st));
        break;
      case GRAB_ARR_BOUNDARIES:
        if (!ix.built) throw Error(GRAB_ERR_STATE, "never built");
        std::memcpy(out, ix.h_bound.data(), (ix.m + 1) * 4);
        break;
      case GRAB_ARR_B2I_OFFSETS: {
        if (!ix.built) throw Error(GRAB_ERR_STATE, "never built");
        uint64_t* o = (uint64_t*)out;
        o[0] = 0;
        for (uint32_t b = 0; b < ix.m; ++b) o[b + 1] = o[b] + ix.h_bcount[b];
        break;
      }
      case GRAB_ARR_B2I_FLAT: {
        if (!ix.built) throw Error(GRAB_ERR_STATE, "never built");
        // members of bucket b = attr[bstart[b] + j].slot, j < bcount[b]
        std::vector<Attr> a(ix.phys_cap);
        GRAB_CUDA(cudaMemcpyAsync(a.data(), ix.attr, ix.phys_cap * sizeof(Attr), cudaMemcpyDeviceToHost, st));
        GRAB_CUDA(cudaStreamSynchronize(st));
        uint32_t* o = (uint32_t*)out;
        uint64_t k = 0;
        for (uint32_t b = 0; b < ix.m; ++b)
          for (uint32_t j = 0; j < ix.h_bcount[b]; ++j) o[k++] = a[ix.h_bstart[b] + j].slot;
        break;
      }
      default:
        throw Error(GRAB_ERR_VALUE, "unknown array selector");
    }
    GRAB_CUDA(cudaStreamSynchronize(st));
  });
}

extern "C" int grab_build(grab_index* h, const float* vectors, const float* scalars, uint64_t n, int strategy,
                          uint32_t k_g, uint32_t refine_rounds, uint32_t mem, grab_build_report* report) {
  return guarded([&] {
    check_handle(h);
    WriteLock lk(h);
    DevIndex& ix = h->ix;
    set_device(ix);
    ix.adj_version++;
    build_index_device(ix, vectors, scalars, n, strategy, k_g, refine_rounds, mem, report);
    ix.adj_version++;
  });
}

extern "C" int grab_build_ex(grab_index* h, const float* vectors, const float* scalars, uint64_t n, int strategy,
                             uint32_t k_g, uint32_t refine_rounds, uint32_t mem, grab_build_report* report,
                             const grab_build_debug* debug) {
  return guarded([&] {
    check_handle(h);
    WriteLock lk(h);
    DevIndex& ix = h->ix;
    set_device(ix);
    ix.adj_version++;
    build_index_device(ix, vectors, scalars, n, strategy, k_g, refine_rounds, mem, report, debug);
    ix.adj_version++;
  });
}

extern "C" int grab_build_graph(grab_index* h, uint32_t k_g, uint32_t refine_rounds, uint64_t exact_limit,
                                uint32_t flags, grab_build_report* report, const grab_build_debug* debug) {
  return guarded([&] {
    check_handle(h);
    WriteLock lk(h);
    DevIndex& ix = h->ix;
    set_device(ix);
    if (!ix.built) throw Error(GRAB_ERR_STATE, "index has no rows / bucket metadata (import first)");
    if (ix.params.k_max > 64) throw Error(GRAB_ERR_VALUE, "k_max > 64 not supported");
    if ((flags & 3) == 3) throw Error(GRAB_ERR_VALUE, "local-only and global-only are exclusive");
    const uint64_t n = ix.count;
    if (k_g == 0) k_g = ix.params.k_max;
    grab_build_report rep{};
    rep.n = n;
    rep.m = ix.m;
    // exact_limit (builder.py:364-393): exact kNN iff n <= exact_limit, else NN-descent
    const uint32_t gp = ix.params.global_pass;
    ix.params.global_pass = n <= exact_limit ? GRAB_GLOBAL_EXACT : GRAB_GLOBAL_DESCENT;
    ix.adj_version++;
    try {
      if (n >= 2 || (flags & kGraphLocalOnly))
        build_graph_device(ix, n, k_g, refine_rounds, &rep, debug, ix.stream, flags);
    } catch (...) {
      ix.params.global_pass = gp;
      throw;
    }
    ix.params.global_pass = gp;
    ix.adj_version++;
    GRAB_CUDA(cudaStreamSynchronize(ix.stream));
    if (report) *report = rep;
  });
}

extern "C" int grab_fuse(grab_index* h, const uint32_t* necessary, const uint32_t* global_rows, uint32_t k_g) {
  return guarded([&] {
    check_handle(h);
    WriteLock lk(h);
    DevIndex& ix = h->ix;
    set_device(ix);
    if (!ix.built) throw Error(GRAB_ERR_STATE, "index has no rows / bucket metadata (import first)");
    if (!necessary || !global_rows || k_g == 0) throw Error(GRAB_ERR_VALUE, "null fuse inputs");
    for (uint64_t i = 0; i < ix.count; ++i)
      if (necessary[i] > ix.params.k_max) throw Error(GRAB_ERR_VALUE, "necessary count > k_max");
    ix.adj_version++;
    if (ix.count) fuse_device(ix, ix.count, necessary, global_rows, k_g);
    ix.adj_version++;
  });
}

extern "C" int grab_reinforce(grab_index* h, uint64_t* added) {
  return guarded([&] {
    check_handle(h);
    WriteLock lk(h);
    DevIndex& ix = h->ix;
    set_device(ix);
    ix.adj_version++;
    const uint32_t a = ix.built ? reinforce_index_device(ix) : 0;
    ix.adj_version++;
    if (added) *added = a;
  });
}

extern "C" int grab_insert(grab_index* h, const float* vectors, const float* scalars, const int64_t* ids, uint64_t b,
                           uint32_t search_itopk, uint32_t mem, grab_insert_report* report) {
  return guarded([&] {
    check_handle(h);
    WriteLock lk(h);
    DevIndex& ix = h->ix;
    set_device(ix);
    ix.adj_version++;
    insert_batch_device(ix, vectors, scalars, ids, b, search_itopk, mem, report);
    ix.adj_version++;
  });
}

extern "C" int grab_append(grab_index* h, const float* vectors, const float* scalars, const int64_t* ids, uint64_t b,
                           uint32_t mem, uint64_t* start, uint64_t* end) {
  return guarded([&] {
    check_handle(h);
    WriteLock lk(h);
    DevIndex& ix = h->ix;
    set_device(ix);
    ix.adj_version++;
    append_batch_device(ix, vectors, scalars, ids, b, mem, start, end);
    ix.adj_version++;
  });
}

extern "C" int grab_last_rewired(const grab_index* h, uint32_t* out, uint64_t cap, uint64_t* n_out) {
  return guarded([&] {
    check_handle(h);
    const auto& v = h->ix.last_rewired;
    if (n_out) *n_out = v.size();
    if (out) std::memcpy(out, v.data(), std::min<uint64_t>(cap, v.size()) * 4);
  });
}

extern "C" int grab_select_neighbors(const float* X, uint64_t n_rows, uint32_t dim, int64_t target,
                                     const int64_t* cand_slots, const double* cand_dists, const uint8_t* cand_fresh,
                                     uint32_t n_cand, uint32_t row_capacity, double alpha, int64_t* out_accepted,
                                     uint32_t* n_accepted) {
  return guarded([&] {
    select_neighbors_device(X, n_rows, dim, target, cand_slots, cand_dists, cand_fresh, n_cand, row_capacity, alpha,
                            out_accepted, n_accepted);
  });
}

extern "C" int grab_try_rewire(const float* X, uint64_t n_rows, uint32_t dim, uint32_t* row, uint32_t k_max,
                               uint32_t v, uint32_t q, double sq_dvq, double alpha, uint32_t k_local,
                               int32_t* accepted, int32_t* evicted_pos) {
  return guarded([&] {
    try_rewire_device(X, n_rows, dim, row, k_max, v, q, sq_dvq, alpha, k_local, accepted, evicted_pos);
  });
}

// ---- stateless helpers -------------------------------------------------------
static DevIndex scratch_view(const float* boundaries, uint32_t m, cudaStream_t st, DBuf& keep) {
  DevIndex v;
  new (&keep) DBuf((m + 1) * 4, st);
  GRAB_CUDA(cudaMemcpyAsync(keep.p, boundaries, (m + 1) * 4, cudaMemcpyHostToDevice, st));
  v.bound = keep.as<float>();
  v.m = m;
  return v;
}

extern "C" int grab_bucket_ids_raw(const float* boundaries, uint32_t m, const float* scalars, uint64_t n,
                                   int32_t* out) {
  return guarded([&] {
    if (m < 1) throw Error(GRAB_ERR_VALUE, "need m >= 1");
    if (!n) return;
    cudaStream_t st = 0;
    DBuf kb;
    DevIndex v = scratch_view(boundaries, m, st, kb);
    DBuf a, c;
    const float* s = stage_in(scalars, n, GRAB_MEM_HOST, a, st);
    int32_t* o = stage_out(out, n, GRAB_MEM_HOST, c, st);
    launch_bucket_ids(v, s, n, o, st);
    copy_back(out, c, n, GRAB_MEM_HOST, st);
    GRAB_CUDA(cudaStreamSynchronize(st));
  });
}

extern "C" int grab_bucket_select_raw(const float* boundaries, uint32_t m, const double* lower, const double* upper,
                                      uint64_t n, int32_t* out_lo, int32_t* out_hi) {
  return guarded([&] {
    if (m < 1) throw Error(GRAB_ERR_VALUE, "need m >= 1");
    if (!n) return;
    cudaStream_t st = 0;
    DBuf kb;
    DevIndex v = scratch_view(boundaries, m, st, kb);
    DBuf a, b, c, d;
    const double* lo = stage_in(lower, n, GRAB_MEM_HOST, a, st);
    const double* hi = stage_in(upper, n, GRAB_MEM_HOST, b, st);
    int32_t* ol = stage_out(out_lo, n, GRAB_MEM_HOST, c, st);
    int32_t* oh = stage_out(out_hi, n, GRAB_MEM_HOST, d, st);
    launch_bucket_select(v, lo, hi, n, ol, oh, st);
    copy_back(out_lo, c, n, GRAB_MEM_HOST, st);
    copy_back(out_hi, d, n, GRAB_MEM_HOST, st);
    GRAB_CUDA(cudaStreamSynchronize(st));
  });
}

namespace grab {
void reverse_merge_raw(const float* X, uint64_t n, uint32_t dim, const uint32_t* graph, uint32_t k, uint32_t k_g,
                       uint32_t* out);  // build.cu
}

extern "C" int grab_reverse_merge_raw(int device, const float* X, uint64_t n, uint32_t dim, const uint32_t* graph,
                                      uint32_t k, uint32_t k_g, uint32_t* out) {
  return guarded([&] {
    if (dim < 1 || k_g < 1) throw Error(GRAB_ERR_VALUE, "dim and k_g must be >= 1");
    if (n >= 0xFFFFFFFFull) throw Error(GRAB_ERR_VALUE, "n exceeds the u32 id space");
    GRAB_CUDA(cudaSetDevice(device));
    if (n) reverse_merge_raw(X, n, dim, graph, k, k_g, out);
  });
}

extern "C" int grab_sq_distances(const float* q, const float* rows, uint64_t n, uint32_t dim, double* out) {
  return guarded([&] {
    if (!n) return;
    if (dim < 1) throw Error(GRAB_ERR_VALUE, "dim must be >= 1");
    cudaStream_t st = 0;
    uint32_t dp = (dim + 3) / 4 * 4;
    DBuf dq(dp * 4, st), dr(n * dp * 4, st), dout(n * 8, st);
    GRAB_CUDA(cudaMemsetAsync(dq.p, 0, dp * 4, st));
    GRAB_CUDA(cudaMemsetAsync(dr.p, 0, n * dp * 4, st));
    GRAB_CUDA(cudaMemcpyAsync(dq.p, q, dim * 4, cudaMemcpyHostToDevice, st));
    GRAB_CUDA(cudaMemcpy2DAsync(dr.p, dp * 4, rows, dim * 4, dim * 4, n, cudaMemcpyHostToDevice, st));
    run_sq_distances(dq.as<float>(), dr.as<float>(), n, dp, dout.as<double>(), st);
    GRAB_CUDA(cudaMemcpyAsync(out, dout.p, n * 8, cudaMemcpyDeviceToHost, st));
    GRAB_CUDA(cudaStreamSynchronize(st));
  });
}

extern "C" int grab_derive_seeds(uint64_t base, const uint32_t* ordinals, uint64_t n, uint64_t* out) {
  return guarded([&] {
    for (uint64_t i = 0; i < n; ++i) out[i] = derive_query_seed(base, ordinals[i]);
  });
}

namespace grab {
uint64_t scc_count_device(const uint32_t* adj, uint32_t n, uint32_t K, cudaStream_t st);  // scc.cu
}

extern "C" int grab_scc_count(const grab_index* h, uint64_t live_count, uint64_t* out) {
  return guarded([&] {
    check_handle(h);
    ReadLock rl(h);
    const DevIndex& ix = h->ix;
    set_device(ix);
    const uint64_t n = live_of(ix, live_count);
    if (n >= 0xFFFFFFFFull) throw Error(GRAB_ERR_VALUE, "too many rows");
    cudaStream_t st = ix.stream;
    DBuf a(std::max<uint64_t>(n, 1) * ix.params.k_max * 4, st);
    adjacency_phys_to_slot(ix, a.as<uint32_t>(), 0, n);
    *out = scc_count_device(a.as<uint32_t>(), (uint32_t)n, ix.params.k_max, st);
  });
}

extern "C" int grab_scc_count_raw(const uint32_t* adjacency, uint64_t rows, uint32_t k_max, uint64_t live_count,
                                  uint64_t* out) {
  return guarded([&] {
    const uint64_t n = std::min(rows, live_count);
    if (n >= 0xFFFFFFFFull) throw Error(GRAB_ERR_VALUE, "too many rows");
    cudaStream_t st = nullptr;
    DBuf a(std::max<uint64_t>(n, 1) * k_max * 4, st);
    GRAB_CUDA(cudaMemcpyAsync(a.p, adjacency, n * k_max * 4, cudaMemcpyHostToDevice, st));
    *out = scc_count_device(a.as<uint32_t>(), (uint32_t)n, k_max, st);
  });
}
