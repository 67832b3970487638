// Host-side entry points of the kernel families (one .cu each).
#pragma once
#include "index.cuh"

namespace grab {

// bruteforce.cu
void run_bruteforce(const DevIndex& ix, const float* Q, uint64_t nq, const double* lo, const double* hi,
                    uint64_t stride, uint32_t k, uint64_t n_live, int64_t* os, double* od, uint32_t* oc,
                    cudaStream_t st);
void run_sq_distances(const float* q, const float* rows, uint64_t n, uint32_t dp, double* out, cudaStream_t st);
// build.cu
void build_index_device(DevIndex& ix, const float* vectors, const float* scalars, uint64_t n, int strategy,
                        uint32_t k_g, uint32_t refine_rounds, uint32_t mem, grab_build_report* report,
                        const grab_build_debug* dbg = nullptr);
// the graph phases on an index whose rows / bucket maps are already in place
// (imported state): pass 1, pass 2, fuse, repair; flags select a subset
constexpr uint32_t kGraphLocalOnly = 1;   // pass 1 only (build_local_phase, builder.py:237-261)
constexpr uint32_t kGraphGlobalOnly = 2;  // pass 2 only (build_global_graph, builder.py:364-393)
void build_graph_device(DevIndex& ix, uint64_t n, uint32_t k_g, uint32_t refine_rounds, grab_build_report* rep,
                        const grab_build_debug* dbg, cudaStream_t st, uint32_t flags);
// fuse_remote_edges (builder.py:396-452) on the imported draft rows; host slot-space inputs
void fuse_device(DevIndex& ix, uint64_t n, const uint32_t* necessary, const uint32_t* global_rows, uint32_t k_g);
// reinforce_reachability (builder.py:455-500) over the live rows; returns links added
uint32_t reinforce_index_device(DevIndex& ix);
// insert.cu
void insert_batch_device(DevIndex& ix, const float* vectors, const float* scalars, const int64_t* ids, uint64_t b,
                         uint32_t search_itopk, uint32_t mem, grab_insert_report* report);
void select_neighbors_device(const float* X, uint64_t n_rows, uint32_t dim, int64_t target, const int64_t* cand_slots,
                             const double* cand_dists, const uint8_t* cand_fresh, uint32_t n_cand,
                             uint32_t row_capacity, double alpha, int64_t* out_accepted, uint32_t* n_accepted);
void try_rewire_device(const float* X, uint64_t n_rows, uint32_t dim, uint32_t* row, uint32_t k_max, uint32_t v,
                       uint32_t q, double sq_dvq, double alpha, uint32_t k_local, int32_t* accepted,
                       int32_t* evicted_pos);

}  // namespace grab
