// solver.h -- power-iteration solver object and its device control block.
#pragma once
#include <cuda_runtime.h>

#include <vector>

#include "plan_impl.h"

namespace tc {

// Device-resident loop state, read by every kernel of an iteration and updated by the last block.
struct Ctrl {
    double c;           // damping (PageRank) / c of Eq. 9 (RWR)
    double tele;        // additive term of the current iteration: PageRank c*D/n + (1-c)/n; RWR 0
    double residual;    // L1 change of the last completed iteration
    double norm[2];     // HITS: norms of the two halves of the last SpMV
    double dmass;       // PageRank: dangling mass of the last iterate
    double tol;
    double inv_n;
    double uniform;     // HITS: value of a zero half after normalisation (reading R5)
    int32_t iter;
    int32_t done;
    uint32_t ticket;
    int32_t max_iter;
    int32_t fixed_iters;
    int32_t q;          // RWR query, relabelled
    double pad_[2];
};

}  // namespace tc

struct spmv_solver_s {
    int algo = 0;
    int64_t n = 0;          // vertices
    int64_t N = 0;          // vector length (n, or 2n for HITS)
    int device = 0;
    spmv_iter_opts it{};
    spmv_plan_s* plan = nullptr;
    std::vector<int32_t> pi;        // original index -> relabelled
    int64_t n_dangling = 0;
    float* d_p = nullptr;           // PageRank p / RWR r / HITS [a;h] (relabelled)
    float* d_y = nullptr;           // partial y (multi-tile rows) / HITS raw product
    float* d_z[2] = {nullptr, nullptr};  // PageRank / RWR SpMV input, double buffered
    float* d_inv = nullptr;         // 1 / (out)degree, 0 for dangling
    uint8_t* d_half = nullptr;      // HITS: 1 for hub entries (vertex order)
    // entry-ordered epilogue state (index = the row's FINAL entry in the plan's row_id[])
    float* d_p_e = nullptr;         // PageRank p / RWR r
    float* d_inv_e = nullptr;       // 1 / degree
    uint8_t* d_half_e = nullptr;    // HITS half flag
    int32_t* d_fpos = nullptr;      // row -> FINAL entry index
    std::vector<int32_t> fpos;      // host copy
    tc::Ctrl* d_ctrl = nullptr;
    double* d_slots = nullptr;
    double pred_extra_us = 0.0;          // model terms beside the plan's SpMV (HITS normalisation)
    std::vector<int> grids;
    std::vector<int32_t> tiles_used, slot_base;
    int32_t total_slots = 0;
    int norm_grid = 0;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    cudaStream_t own_stream = nullptr;
    tc::Ctrl last{};
    spmv_comm comm = nullptr;       // multi-GPU solvers (dist.cu)
    void* batch = nullptr;          // batched RWR state (batch.cu)
    void* dist = nullptr;
};

// multi-GPU row-partitioned solvers (dist.cu)
struct LocalInput {                 // spmv_solver_create_local: this rank's rows only
    int64_t n_local;
    const int32_t* owned;           // [n_local] global vertex ids
    const int64_t* row_ptr;         // [n_local + 1] rows of the iteration matrix
    const int32_t* col;             // global column ids
    const int32_t* out_degree;      // [n_local] (PageRank); NULL: the row length (RWR)
};
spmv_status solver_create_dist(int algo, int64_t n, int64_t m, const int64_t* row_ptr,
                               const int32_t* col, const spmv_iter_opts* it,
                               const spmv_options* opt, spmv_comm comm, int device,
                               spmv_solver* out, const LocalInput* li = nullptr);
spmv_status solver_run_dist(spmv_solver s, int64_t query, void* stream, spmv_iter_result* res);
spmv_status solver_result_dist(spmv_solver s, float* out0, float* out1);
void solver_destroy_dist(spmv_solver s);
void batch_destroy(spmv_solver s);
