// launch.cuh -- the tile launcher shared by spmv_execute and the power iterations.
#pragma once
#include <algorithm>
#include <vector>

#include "plan_impl.h"
#include "tc_kernels.cuh"

namespace tc {

void set_error(const std::string& msg);
spmv_status cuda_status(cudaError_t e, const char* what);

// Kernel launch, with programmatic stream serialization when `pdl` (the kernel's
// griddepcontrol.wait then orders it after the previous launch on the stream).
template <class... Args>
cudaError_t launch_k(void (*k)(Args...), int grid, int block, size_t smem, cudaStream_t st, bool pdl,
                     Args... args) {
    if (!pdl) { k<<<grid, block, smem, st>>>(args...); return cudaGetLastError(); }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid); cfg.blockDim = dim3((unsigned)block);
    cfg.dynamicSmemBytes = smem; cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k, args...);
}

// Launch tile t of `p` (x given relabelled: xp[k] = x[perm[k]]).  pdl: chained to the previous
// launch on the stream by programmatic dependent launch (standalone products).
template <class Epi>
cudaError_t launch_tile(const spmv_plan_s& p, int32_t t, int grid, const float* xp,
                        const Epi& epi, cudaStream_t st, bool pdl = false) {
    const TileInfo& ti = p.tiles[t];
    TileArgs a;
    a.desc = p.d_desc; a.wl_begin = ti.wl_begin; a.wl_end = ti.wl_end;
    a.col = p.d_col; a.val = p.d_val; a.row_id = p.d_row_id;
    a.x = xp + ti.col_lo; a.width = (int32_t)(ti.col_hi - ti.col_lo);
    a.split = p.d_split; a.partials = p.d_partials; a.counters = p.d_counters;
    a.sched = p.d_sched + (kDynQ + 1) * t;
    a.has_acc = t > 0;                     // the first tile's rows are all first touches
    if (!a.has_acc) {                      // first touches only: FirstTouch<Epi> (tc_kernels.cuh)
        const FirstTouch<Epi> ft(epi);
        if (ti.staged) {
            size_t smem = (size_t)a.width * sizeof(float);
            if (p.pattern) return launch_k(tc_spmv_tile<true, false, FirstTouch<Epi>>, grid, kThreads, smem, st, pdl, a, ft);
            return launch_k(tc_spmv_tile<true, true, FirstTouch<Epi>>, grid, kThreads, smem, st, pdl, a, ft);
        }
        if (p.pattern) return launch_k(tc_spmv_tile<false, false, FirstTouch<Epi>>, grid, kThreads, 0, st, pdl, a, ft);
        return launch_k(tc_spmv_tile<false, true, FirstTouch<Epi>>, grid, kThreads, 0, st, pdl, a, ft);
    }
    if (ti.staged) {
        size_t smem = (size_t)a.width * sizeof(float);
        if (p.pattern) return launch_k(tc_spmv_tile<true, false, Epi>, grid, kThreads, smem, st, pdl, a, epi);
        return launch_k(tc_spmv_tile<true, true, Epi>, grid, kThreads, smem, st, pdl, a, epi);
    }
    if (p.pattern) return launch_k(tc_spmv_tile<false, false, Epi>, grid, kThreads, 0, st, pdl, a, epi);
    return launch_k(tc_spmv_tile<false, true, Epi>, grid, kThreads, 0, st, pdl, a, epi);
}

// Launch every non-empty tile of `p` in ascending order.
template <class Epi>
cudaError_t launch_tiles(const spmv_plan_s& p, const std::vector<int>& grids, const float* xp,
                         const Epi& epi, cudaStream_t st, bool pdl = false) {
    for (int32_t t = 0; t <= p.num_tiles; ++t) {
        if (p.tiles[t].wl_end == p.tiles[t].wl_begin) continue;
        cudaError_t e = launch_tile(p, t, grids[t], xp, epi, st, pdl);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

// Occupancy-derived persistent grids for an epilogue type (called once per plan per Epi).
// Tiles whose x segment cannot be staged (no CTA fits) fall back to the read-only path.
template <class Epi>
cudaError_t setup_grids(spmv_plan_s& p, std::vector<int>& grids) {
    cudaError_t e;
    auto kst = p.pattern ? tc_spmv_tile<true, false, Epi> : tc_spmv_tile<true, true, Epi>;
    auto kgl = p.pattern ? tc_spmv_tile<false, false, Epi> : tc_spmv_tile<false, true, Epi>;
    int optin = 0;
    if ((e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, p.device))) return e;
    cudaFuncAttributes fa;
    if ((e = cudaFuncGetAttributes(&fa, kst))) return e;
    const int max_dyn = optin - (int)fa.sharedSizeBytes;
    if ((e = cudaFuncSetAttribute(kst, cudaFuncAttributeMaxDynamicSharedMemorySize, max_dyn))) return e;
    {   // the first-touch instantiations launched for first tiles (launch_tile)
        auto fst = p.pattern ? tc_spmv_tile<true, false, FirstTouch<Epi>> : tc_spmv_tile<true, true, FirstTouch<Epi>>;
        auto fgl = p.pattern ? tc_spmv_tile<false, false, FirstTouch<Epi>> : tc_spmv_tile<false, true, FirstTouch<Epi>>;
        if ((e = cudaFuncSetAttribute(fst, cudaFuncAttributeMaxDynamicSharedMemorySize, max_dyn))) return e;
        if ((e = cudaFuncSetAttribute(fgl, cudaFuncAttributeMaxDynamicSharedMemorySize, max_dyn))) return e;
    }
    int nb = 0;
    if ((e = cudaFuncSetAttribute(kgl, cudaFuncAttributeMaxDynamicSharedMemorySize, max_dyn))) return e;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kgl, kThreads, 0))) return e;
    const int g_global = std::max(1, nb) * p.sm_count;
    grids.assign(p.num_tiles + 1, g_global);
    for (int32_t t = 0; t <= p.num_tiles; ++t) {
        if (!p.tiles[t].staged) continue;
        size_t smem = (size_t)(p.tiles[t].col_hi - p.tiles[t].col_lo) * sizeof(float);
        if ((int64_t)smem > max_dyn) { p.tiles[t].staged = 0; continue; }
        if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kst, kThreads, smem))) return e;
        if (nb < 1) { p.tiles[t].staged = 0; continue; }
        grids[t] = nb * p.sm_count;
    }
    return cudaSuccess;
}

}  // namespace tc
