/*
 * grab.h -- C ABI of the B200-native GRAB-ANNS range-filtered graph index.
 *
 * The reference (/root/reference/pkg/src/bucketann, pure Python + numpy) has no
 * FFI: callers use the Python functions re-exported by bucketann/__init__.py:3-44.
 * Each entry point below replaces one of those functions; the Python package
 * paper_2604_16402_b200 binds them with ctypes and rebuilds the reference's
 * return types (SearchResult, BuildReport, InsertReport, GraphIndex views).
 *
 * Conventions
 *  - plain pointers + sizes; no torch types.
 *  - ids crossing the ABI are reference SLOT ids (physical row order in the
 *    reference's VectorStore, layout.py:22-79); the device keeps its own
 *    bucket-slab physical order internally.
 *  - `mem` selects where pointer arguments live: GRAB_MEM_HOST (copied by the
 *    library, synchronous) or GRAB_MEM_DEVICE (device pointers, enqueued on
 *    `stream`, asynchronous).
 *  - every call returns GRAB_OK or a GRAB_ERR_* code; grab_last_error() gives
 *    the message (thread-local). Codes map 1:1 to the reference's exceptions
 *    (core.py:17-22, layout.py:59-63,200-207).
 */
#ifndef GRAB_H_
#define GRAB_H_

#include <stdint.h>

#if defined(__GNUC__)
#define GRAB_API __attribute__((visibility("default")))
#else
#define GRAB_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define GRAB_OK 0
#define GRAB_ERR_VALUE 1     /* ValueError */
#define GRAB_ERR_DIMENSION 2 /* DimensionMismatchError (ValueError) */
#define GRAB_ERR_CAPACITY 3  /* CapacityError (RuntimeError) */
#define GRAB_ERR_CUDA 4      /* device failure */
#define GRAB_ERR_STATE 5     /* e.g. operation on a never-built index */

#define GRAB_MEM_HOST 0
#define GRAB_MEM_DEVICE 1

#define GRAB_SENTINEL 0xFFFFFFFFu /* empty adjacency slot, layout.py:19 */
#define GRAB_LIVE_ALL 0xFFFFFFFFFFFFFFFFull

#define GRAB_STRATEGY_QUANTILE 0
#define GRAB_STRATEGY_WIDTH 1

typedef struct grab_index grab_index;

/* BuildParams (core.py:85-118) */
/* global_pass: pass-2 candidate graph (builder.py:379-391) */
#define GRAB_GLOBAL_AUTO 0    /* reference rule: exact kNN iff n <= 100 000, else NN-descent */
#define GRAB_GLOBAL_EXACT 1   /* exact kNN at every n (tcgen05 screen + f64 rerank) */
#define GRAB_GLOBAL_DESCENT 2 /* random init + refine_rounds of neighborhood descent */

typedef struct {
  uint32_t k_max, k_local, bucket_capacity, global_pass;
  double proximal_fraction, proximal_window, alpha;
  uint64_t rng_seed;
} grab_build_params;

/* SearchParams minus the range (core.py:121-147); seed_count 0 = min(itopk, 32) */
typedef struct {
  uint32_t k, itopk, search_width, max_iterations, seed_count, _pad;
} grab_search_params;

/* SearchStats (searcher.py:22-31) + `expanded` (frontier nodes popped) */
typedef struct {
  uint32_t iterations, dist_evals, seed_evals, gathered;
  uint32_t in_range_new, precheck_rejected, seed_attempts, expanded;
} grab_search_stats;

/* BuildReport (builder.py:63-76) */
typedef struct {
  uint64_t n;
  uint32_t m, isolated_nodes;
  double phase1_seconds, phase2_seconds, fuse_seconds, total_seconds;
  double cross_bucket_edge_ratio;
  uint32_t global_descent, _pad; /* 1 when pass 2 ran NN-descent */
} grab_build_report;

/* InsertReport (updater.py:31-46); rewired rows via grab_last_rewired() */
typedef struct {
  uint64_t batch_size, bulk_built, forward_accepted, forward_rejected;
  uint64_t reverse_accepted, reverse_rejected, evictions_necessary, evictions_redundant;
  uint64_t forced_links, n_rewired;
  double wall_time_s;
  /* seconds: append, in-bucket candidates, candidate search, forward selection,
   * reverse rewiring, healing */
  double phase_seconds[6];
} grab_insert_report;

typedef struct {
  uint64_t count, capacity;
  uint32_t dim, k_max, k_local, m;
  int32_t built;
  uint32_t _pad;
  uint64_t phys_capacity, device_bytes;
} grab_info_t;

/* grab_read / grab_write array selectors (slot space unless noted) */
#define GRAB_ARR_X 0          /* f32 [count x dim] */
#define GRAB_ARR_SCALARS 1    /* f32 [count] */
#define GRAB_ARR_ADJ 2        /* u32 [count x k_max], slot ids / SENTINEL */
#define GRAB_ARR_I2B 3        /* i32 [count] (M_I2B) */
#define GRAB_ARR_BOUNDARIES 4 /* f32 [m+1] */
#define GRAB_ARR_B2I_OFFSETS 5 /* u64 [m+1]: bucket b members are B2I_FLAT[off[b]:off[b+1]] */
#define GRAB_ARR_B2I_FLAT 6   /* u32 [count]: M_B2I lists concatenated, insertion order */

/* ---- lifecycle (create_index, layout.py:250-257) ---- */
GRAB_API int grab_create(int device, uint32_t dim, uint64_t capacity, const grab_build_params* params,
                grab_index** out);
GRAB_API void grab_destroy(grab_index* h);
GRAB_API const char* grab_last_error(void);
GRAB_API int grab_get_info(const grab_index* h, grab_info_t* out);
GRAB_API int grab_sync(grab_index* h);

/* ---- build_index (builder.py:503-548) over host or device rows ---- */
GRAB_API int grab_build(grab_index* h, const float* vectors, const float* scalars, uint64_t n, int strategy,
               uint32_t k_g, uint32_t refine_rounds, uint32_t mem, grab_build_report* report);

/* Optional capture of the intermediate graphs (host pointers, slot ids, NULL
 * to skip): pass-1 forward kNN rows and merged rows (LocalGraphDraft,
 * builder.py:38-52), necessary counts, and the pass-2 global rows
 * (GlobalGraph.rows, builder.py:55-60), each [n x k] with k = k_max / k_g. */
typedef struct {
  uint32_t* forward_rows;
  uint32_t* merged_rows;
  uint32_t* necessary;
  uint32_t* global_rows;
} grab_build_debug;
GRAB_API int grab_build_ex(grab_index* h, const float* vectors, const float* scalars, uint64_t n,
                           int strategy, uint32_t k_g, uint32_t refine_rounds, uint32_t mem,
                           grab_build_report* report, const grab_build_debug* debug);

/* ---- the build phases on an imported state (grab_import: rows, scalars,
 * bucket maps; SENTINEL or draft adjacency), for the reference's phase-level
 * API. flags: 0 = pass 1 + pass 2 + fuse + repair (build_index minus the
 * partition), GRAB_GRAPH_LOCAL_ONLY = pass 1 (build_local_phase,
 * builder.py:237-261), GRAB_GRAPH_GLOBAL_ONLY = pass 2 (build_global_graph,
 * builder.py:364-393: exact kNN iff count <= exact_limit, else random init +
 * refine_rounds NN-descent rounds). Intermediate rows via `debug`. */
#define GRAB_GRAPH_LOCAL_ONLY 1
#define GRAB_GRAPH_GLOBAL_ONLY 2
GRAB_API int grab_build_graph(grab_index* h, uint32_t k_g, uint32_t refine_rounds, uint64_t exact_limit,
                              uint32_t flags, grab_build_report* report, const grab_build_debug* debug);
/* fuse_remote_edges (builder.py:396-452): the index adjacency holds the draft
 * rows (imported); necessary [count] and global_rows [count x k_g] are host,
 * slot space. Read the fused rows back with grab_read(GRAB_ARR_ADJ). */
GRAB_API int grab_fuse(grab_index* h, const uint32_t* necessary, const uint32_t* global_rows, uint32_t k_g);
/* reinforce_reachability (builder.py:455-500) on the live rows; *added = links added */
GRAB_API int grab_reinforce(grab_index* h, uint64_t* added);

/* ---- insert_batch (updater.py:154-263) ---- */
GRAB_API int grab_insert(grab_index* h, const float* vectors, const float* scalars, const int64_t* ids,
                uint64_t b, uint32_t search_itopk, uint32_t mem, grab_insert_report* report);
GRAB_API int grab_last_rewired(const grab_index* h, uint32_t* out, uint64_t cap, uint64_t* n_out);
/* append_batch (layout.py:181-223): rows / scalars / ids and bucket maps only
 * (adjacency of the new slots stays SENTINEL); [*start, *end) = the new slots.
 * Needs bucket metadata (a built index). */
GRAB_API int grab_append(grab_index* h, const float* vectors, const float* scalars, const int64_t* ids, uint64_t b,
                         uint32_t mem, uint64_t* start, uint64_t* end);

/* ---- search / search_batch (searcher.py:156-248) ----
 * Query i uses range [lower[i*range_stride], upper[i*range_stride]] (stride 0 =
 * one shared range, as search_batch) and RNG seed seeds[i] when `seeds` is
 * non-NULL, else derive_query_seed(seed_base, ordinal0 + i) (searcher.py:85-87).
 * live_count = GRAB_LIVE_ALL uses the published count. Outputs: k slots
 * (int64, -1 padded) and squared distances (f64) per query, ascending by
 * (dist, slot); out_counts[i] = result length; out_stats optional. */
GRAB_API int grab_search(const grab_index* h, const float* queries, uint64_t nq, const double* lower,
                const double* upper, uint64_t range_stride, const grab_search_params* params,
                const uint64_t* seeds, uint64_t seed_base, uint64_t ordinal0, uint64_t live_count,
                int64_t* out_slots, double* out_dists, uint32_t* out_counts,
                grab_search_stats* out_stats, uint32_t mem, void* stream);

/* ---- brute_force_search (evaluate.py:22-44): exact (dist, slot) top-k ---- */
GRAB_API int grab_brute_force(const grab_index* h, const float* queries, uint64_t nq, const double* lower,
                     const double* upper, uint64_t range_stride, uint32_t k, uint64_t live_count,
                     int64_t* out_slots, double* out_dists, uint32_t* out_counts, uint32_t mem,
                     void* stream);

/* ---- bucket selection: intersecting_buckets / bucket_ids_of (layout.py:157-174) ---- */
GRAB_API int grab_bucket_select(const grab_index* h, const double* lower, const double* upper, uint64_t n,
                       int32_t* out_lo, int32_t* out_hi, uint32_t mem, void* stream);
GRAB_API int grab_bucket_ids(const grab_index* h, const float* scalars, uint64_t n, int32_t* out,
                    uint32_t mem, void* stream);

/* partition_buckets (layout.py:107-154) on `device`: boundaries (np.unique of the
 * quantile / width edges) into out_boundaries (host, capacity max_boundaries >=
 * ceil(n / target_capacity) + 1), *out_m = buckets, and optionally the bucket id
 * of every scalar into out_ids (mem-space like scalars). Stream: the caller's in
 * device mode, the legacy default stream otherwise. */
GRAB_API int grab_partition(int device, const float* scalars, uint64_t n, uint32_t target_capacity, int strategy,
                            float* out_boundaries, uint32_t max_boundaries, uint32_t* out_m, int32_t* out_ids,
                            uint32_t mem, void* stream);

/* stateless variants over explicit boundaries f32[m+1] (host pointers) */
GRAB_API int grab_bucket_ids_raw(const float* boundaries, uint32_t m, const float* scalars, uint64_t n,
                                 int32_t* out);
GRAB_API int grab_bucket_select_raw(const float* boundaries, uint32_t m, const double* lower,
                                    const double* upper, uint64_t n, int32_t* out_lo, int32_t* out_hi);

/* ---- sq_distances (core.py:25-38): f64-accumulated squared L2, host pointers ----
 * Same reduction tree as the search / brute-force kernels (bit-identical). */
GRAB_API int grab_sq_distances(const float* q, const float* rows, uint64_t n, uint32_t dim, double* out);

/* ---- state import / export (GraphIndex <-> device layout; dataio.py:111-187) ---- */
GRAB_API int grab_import(grab_index* h, uint64_t n, const float* X, const float* scalars,
                const uint32_t* adjacency, const float* boundaries, uint32_t m, const int32_t* i2b,
                const uint32_t* b2i_flat, const uint64_t* b2i_offsets);
GRAB_API int grab_read(const grab_index* h, int what, uint64_t start, uint64_t count, void* out);

/* ---- pruning primitives on explicit inputs (updater.py:49-123) ---- */
/* select_neighbors: rows X [n_rows x dim] (host), candidates (slot, f64 dist)
 * sorted ascending; fresh[i] != 0 marks Q_new. Returns accepted slots. */
GRAB_API int grab_select_neighbors(const float* X, uint64_t n_rows, uint32_t dim, int64_t target,
                          const int64_t* cand_slots, const double* cand_dists,
                          const uint8_t* cand_fresh, uint32_t n_cand, uint32_t row_capacity,
                          double alpha, int64_t* out_accepted, uint32_t* n_accepted);
/* try_rewire on one adjacency row (k_max entries, slot ids) */
GRAB_API int grab_try_rewire(const float* X, uint64_t n_rows, uint32_t dim, uint32_t* row, uint32_t k_max,
                    uint32_t v, uint32_t q, double sq_dvq, double alpha, uint32_t k_local,
                    int32_t* accepted, int32_t* evicted_pos);

/* ---- scc_count (evaluate.py:60-119): strongly connected components of the
 * live graph (slot space; SENTINEL and targets >= live_count ignored), counted
 * on the device (trim + forward-max coloring + backward closure). ---- */
GRAB_API int grab_scc_count(const grab_index* h, uint64_t live_count, uint64_t* out);
/* the same over an explicit slot-space adjacency (host pointer, rows x k_max) */
GRAB_API int grab_scc_count_raw(const uint32_t* adjacency, uint64_t rows, uint32_t k_max, uint64_t live_count,
                                uint64_t* out);
/* _reverse_merge_topk (builder.py:338-361) over an explicit graph (host
 * pointers): rows X [n x dim] f32, graph [n x k] slot ids (SENTINEL = none,
 * k <= k_g); union with the reverse edges, dedup, the k_g nearest per row by
 * (f64 distance, slot) -> out [n x k_g] (SENTINEL padded). The kernels of the
 * device build's global pass. */
GRAB_API int grab_reverse_merge_raw(int device, const float* X, uint64_t n, uint32_t dim, const uint32_t* graph,
                                    uint32_t k, uint32_t k_g, uint32_t* out);

/* ---- bucket-range sharded search (no reference counterpart:
 * the reference is single-process, so these replace nothing and follow the
 * reference's result convention -- ascending (distance, slot) with GLOBAL slot
 * ids, searcher.py:64-71). Device pointers, enqueued on `stream`. ----
 * pack: per searched query q = qidx[i] (global query index), its k results
 * (local slots -> gid[slot], -1 kept) go to send[(q / B) * B + q % B][0..k):
 * the block of owner rank q / B. Every other block is filled NaN / -1. */
GRAB_API int grab_shard_pack(uint64_t n, const uint32_t* qidx, const int64_t* slots, const double* dists,
                             const int64_t* gid, uint32_t k, uint32_t world, uint32_t B, double* send_d,
                             int64_t* send_i, void* stream);
/* Fused exchange over peer memory (NVLink): pack straight into every owner's
 * receive buffer [src][B][k] through CUDA IPC mappings. peer_d / peer_i are
 * device arrays of `world` pointers (entry r = rank r's receive buffer, the
 * local one for r == rank); this rank fills its slice [rank] of every owner's
 * buffer with NaN / -1, then stores its results. The caller synchronizes the
 * ranks (stream sync + barrier) before grab_merge_topk. */
GRAB_API int grab_shard_pack_p2p(uint64_t n, const uint32_t* qidx, const int64_t* slots, const double* dists,
                                 const int64_t* gid, uint32_t k, uint32_t rank, uint32_t world, uint32_t B,
                                 double* const* peer_d, int64_t* const* peer_i, void* stream);
/* The same exchange without any host synchronisation: stream-ordered peer flags.
 * Each rank owns an IPC-shareable sync block of grab_shard_sync_bytes(world)
 * bytes, zeroed once (my_sync; peer_sync = device array of every rank's block,
 * the local one for r == rank), and numbers its batches epoch = 1, 2, ...
 * identically on every rank. pack_p2p_sync: waits on the device until every
 * owner has merged batch epoch - 1, writes every entry of this rank's slice of
 * every owner's buffer (results of the nq-query batch's routed subset, empty
 * elsewhere), then publishes `epoch` into every owner's ready word for this
 * rank. merge_topk_p2p: waits on the device until all world ready words reach
 * `epoch`, merges, then publishes `epoch` into every rank's free word for this
 * owner. inv_scratch: nq int32 of device scratch. */
GRAB_API uint64_t grab_shard_sync_bytes(uint32_t world);
GRAB_API int grab_shard_pack_p2p_sync(uint32_t nq, uint64_t n, const uint32_t* qidx, const int64_t* slots,
                                      const double* dists, const int64_t* gid, uint32_t k, uint32_t rank,
                                      uint32_t world, uint32_t B, double* const* peer_d, int64_t* const* peer_i,
                                      uint64_t* my_sync, uint64_t* const* peer_sync, uint64_t epoch,
                                      int32_t* inv_scratch, void* stream);
GRAB_API int grab_merge_topk_p2p(uint32_t nq, uint32_t nsrc, uint32_t B, uint32_t k, const double* d,
                                 const int64_t* id, double* out_d, int64_t* out_i, uint32_t* out_c, uint32_t rank,
                                 uint64_t* my_sync, uint64_t* const* peer_sync, uint64_t epoch, void* stream);
/* IPC-shareable device buffers: allocate (zero-filled, 64-byte handle out), open a peer's, close, free */
GRAB_API int grab_ipc_alloc(uint64_t bytes, void** ptr, void* handle64);
GRAB_API int grab_ipc_open(const void* handle64, void** ptr);
GRAB_API int grab_ipc_close(void* ptr);
GRAB_API int grab_ipc_free(void* ptr);
/* derive_query_seed(base, ordinals[i]) for a routed subset of a batch
 * (searcher.py:85-87; host pointers) */
GRAB_API int grab_derive_seeds(uint64_t base, const uint32_t* ordinals, uint64_t n, uint64_t* out);
/* merge: recv[src][B][k] (after the all-to-all) -> per owned query the top-k of
 * the nsrc lists by (distance, global id); out_c = result length. */
GRAB_API int grab_merge_topk(uint32_t nq, uint32_t nsrc, uint32_t B, uint32_t k, const double* d,
                             const int64_t* id, double* out_d, int64_t* out_i, uint32_t* out_c, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* GRAB_H_ */
