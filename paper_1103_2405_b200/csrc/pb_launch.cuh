// pb_launch.cuh -- launcher of the two-phase tiles (pb_kernels.cuh), shared by spmv_execute and
// the power iterations.
#pragma once
#include <algorithm>

#include "pb_kernels.cuh"
#include "plan_impl.h"

namespace tc {

inline PbArgs pb_args(const spmv_plan_s& p, const float* x) {
    PbArgs a;
    a.items = p.d_pb_items; a.runs = p.d_pb_runs; a.cd = p.d_pb_cd;
    a.val = p.pattern ? nullptr : p.d_pb_val; a.pos = p.d_pb_pos; a.prow = p.d_row_id;
    a.pmeta = p.d_pb_pmeta; a.group_chunks = p.d_pb_gchunks;
    a.n_items = (int32_t)p.PB.items.size(); a.n_groups = p.pb_groups;
    a.buf = p.d_pb_buf; a.x = x; a.ctl = p.d_pb_ctl;
    a.n_cols = p.n_cols;
    a.stage_bytes = (int32_t)p.PB.stage_bytes;
    a.trace = nullptr;
    return a;
}

// persistent grid of the Epi instantiation: resident CTAs per SM x SMs
template <class Epi>
cudaError_t pb_setup(const spmv_plan_s& p, int& grid) {
    auto k = p.pattern ? pb_spmv<false, Epi> : pb_spmv<true, Epi>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.pb_smem);
    if (e) return e;
    int nb = 0;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, kPbThreads, (size_t)p.pb_smem))) return e;
    grid = std::max(1, nb) * p.sm_count;
    return cudaSuccess;
}

template <class Epi>
cudaError_t launch_pb(const spmv_plan_s& p, int grid, const float* x, const Epi& epi, cudaStream_t st,
                      int64_t* trace = nullptr) {
    PbArgs a = pb_args(p, x);
    a.trace = trace;
    // cooperative: every CTA of the persistent grid is resident (a reduce waits for expands that
    // other CTAs own)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid); cfg.blockDim = dim3(kPbThreads);
    cfg.dynamicSmemBytes = (size_t)p.pb_smem; cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative; at[0].val.cooperative = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    if (p.pattern) return cudaLaunchKernelEx(&cfg, pb_spmv<false, Epi>, a, epi);
    return cudaLaunchKernelEx(&cfg, pb_spmv<true, Epi>, a, epi);
}

}  // namespace tc
