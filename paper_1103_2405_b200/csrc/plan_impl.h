// plan_impl.h -- the plan object behind spmv_plan, and the tile launcher shared by
// spmv_execute and the power iterations.
#pragma once
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "pb.h"
#include "plan.h"

struct spmv_plan_s {
    int64_t n_rows = 0, n_cols = 0, nnz = 0;
    bool pattern = false;
    int device = -1;
    spmv_options opt{};
    tc::HostLayout L;              // host copy (kept for host-only plans; fetched on demand)
    bool host_valid = false;
    std::vector<int32_t> perm;
    int32_t num_tiles = 0, tile_width = 0;
    int64_t n_workloads = 0, n_slots = 0, n_row_entries = 0, n_split = 0, n_chunks = 0;
    std::vector<tc::TileInfo> tiles;
    double predicted_us = 0.0, build_ms = 0.0;
    int32_t perf_table_loaded = 0;
    int32_t orient = 0;                 // workload orientation in use (the model's choice for -1)
    // device
    tc::WlDesc* d_desc = nullptr;
    uint32_t* d_row_id = nullptr;
    int32_t* d_col = nullptr;
    float* d_val = nullptr;
    int32_t* d_perm = nullptr;
    int32_t* d_inv = nullptr;           // inverse relabel (scatter form of the x permutation)
    bool permute_gather = true;         // x'[k] = x[perm[k]]; TCSPMV_PERMUTE=scatter: x'[inv[j]] = x[j]
    float* d_xp = nullptr;          // relabelled x for spmv_execute
    float* d_hx = nullptr;          // spmv_execute_host staging (x then y)
    float* d_hxb = nullptr;         // spmv_execute_host_batch: kPipe (x, y) buffer pairs
    cudaStream_t s_h2d = nullptr, s_d2h = nullptr;  // its copy streams
    static constexpr int kPipe = 3;
    cudaEvent_t ev_pipe[3 * kPipe + 2] = {};   // h2d done[kPipe], compute done[kPipe], d2h done[kPipe], start, end
    int32_t* d_split = nullptr;
    float* d_partials = nullptr;
    int32_t* d_counters = nullptr;
    uint32_t* d_sched = nullptr;    // [(kDynQ + 1) * (num_tiles + 1)] dynamic-schedule counters
    int64_t device_bytes = 0;
    int sm_count = 0;
    std::vector<int> grid_tile;     // per tile persistent grid for EpiStore
    // two-phase tiles (pb.h): when set, the plan has no one-pass tiles; d_row_id holds the
    // two-phase row order (row | FLAG_FINAL, n_row_entries = n_rows) for the epilogues
    bool two_phase = false;
    bool pdl = false;                   // standalone launches chained by programmatic dependent launch
    tc::PbLayout PB;                      // host copy; the per-entry arrays are released after upload
    bool pb_host_valid = false;
    int32_t* d_pb_runs = nullptr;
    uint32_t* d_pb_cd = nullptr;
    float* d_pb_val = nullptr;
    uint16_t* d_pb_pos = nullptr;
    uint32_t* d_pb_pmeta = nullptr;
    tc::PbItem* d_pb_items = nullptr;
    int32_t* d_pb_gchunks = nullptr;
    float* d_pb_buf = nullptr;
    uint32_t* d_pb_ctl = nullptr;
    int64_t pb_smem = 0;
    int pb_grid = 0;                      // persistent grid of the EpiStore instantiation
    int64_t pb_chunks = 0, pb_bins = 0, pb_long = 0;
    int32_t pb_groups = 0;
    double one_pass_us = 0.0, two_phase_us = 0.0;
    // plan-owned scratch (d_xp, split partials and counters, claim queues) is used by one
    // product at a time: a product on another stream than the previous one waits for it
    cudaEvent_t ev_scratch = nullptr;
    cudaStream_t scratch_stream = nullptr;
    bool scratch_used = false;
};

namespace tc {
spmv_status cuda_status(cudaError_t e, const char* what);
// build the plan (host) and upload it to `device` (capi.cu)
spmv_status plan_final_positions(spmv_plan_s* p, std::vector<uint32_t>& entries, std::vector<int32_t>& fpos);
spmv_status create_plan(int64_t n_rows, int64_t n_cols, int64_t nnz, const int64_t* row_ptr,
                        const int32_t* col, const float* val, const spmv_options* opt_in,
                        int device, spmv_plan_s** out);
}  // namespace tc
