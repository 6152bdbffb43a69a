// launch.cuh -- the tile launcher shared by spmv_execute and the power iterations.
#pragma once
#include <algorithm>
#include <vector>

#include "plan_impl.h"
#include "tc_kernels.cuh"

namespace tc {

void set_error(const std::string& msg);
spmv_status cuda_status(cudaError_t e, const char* what);

// streaming geometry of tile t: warps per CTA limited by shared memory (x segment + two
// buffers per warp); false if not even one warp fits
inline bool ws_geometry(const spmv_plan_s& p, int32_t t, bool staged, WsArgs& s, size_t& smem, int& threads) {
    const TileInfo& ti = p.tiles[t];
    const int64_t width = ti.col_hi - ti.col_lo;
    s.x_floats = staged ? (int32_t)((width + 3) / 4 * 4) : 0;
    s.buf_slots = p.stage_slots;
    const int64_t per_warp = 2LL * s.buf_slots * 4 * (p.pattern ? 1 : 2);
    const int64_t avail = (int64_t)p.max_dyn_smem - ws_bar_bytes(16) - (int64_t)s.x_floats * 4;
    int64_t nw = std::min<int64_t>(kStreamThreads / 32, avail / per_warp);
    if (nw < 4) return false;
    threads = (int)nw * 32;
    smem = (size_t)ws_bar_bytes((int)nw) + (size_t)s.x_floats * 4 + (size_t)nw * per_warp;
    return true;
}

// Launch tile t of `p` (x given relabelled: xp[k] = x[perm[k]]).
template <class Epi>
cudaError_t launch_tile(const spmv_plan_s& p, int32_t t, int grid, const float* xp,
                        const Epi& epi, cudaStream_t st) {
    const TileInfo& ti = p.tiles[t];
    TileArgs a;
    a.desc = p.d_desc; a.wl_begin = ti.wl_begin; a.wl_end = ti.wl_end;
    a.col = p.d_col; a.val = p.d_val; a.row_id = p.d_row_id;
    a.x = xp + ti.col_lo; a.width = (int32_t)(ti.col_hi - ti.col_lo);
    a.hot = p.l1_hot_cols;
    a.prefix = ti.staged ? 0 : (int32_t)std::min<int64_t>(p.x_prefix, ti.col_hi - ti.col_lo);
    a.split = p.d_split; a.partials = p.d_partials; a.counters = p.d_counters;
    a.sched = p.d_sched + (kDynQ + 1) * t;
    if (p.stream) {
        WsArgs s;
        size_t smem = 0;
        int threads = 0;
        bool staged = ti.staged != 0;
        bool fits = true;
        if (staged && !ws_geometry(p, t, true, s, smem, threads)) staged = false;
        if (!staged && !ws_geometry(p, t, false, s, smem, threads)) fits = false;
        if (!fits) {
            // workloads too large for per-warp buffers: this tile runs the classic kernel
        } else if (staged) {
            if (p.pattern) tc_spmv_wstream<true, false, Epi><<<p.stream_grid, threads, smem, st>>>(a, s, epi);
            else tc_spmv_wstream<true, true, Epi><<<p.stream_grid, threads, smem, st>>>(a, s, epi);
        } else {
            if (p.pattern) tc_spmv_wstream<false, false, Epi><<<p.stream_grid, threads, smem, st>>>(a, s, epi);
            else tc_spmv_wstream<false, true, Epi><<<p.stream_grid, threads, smem, st>>>(a, s, epi);
        }
        if (fits) return cudaGetLastError();
    }
    if (ti.staged) {
        size_t smem = (size_t)a.width * sizeof(float);
        if (p.pattern) tc_spmv_tile<true, false, Epi><<<grid, kThreads, smem, st>>>(a, epi);
        else tc_spmv_tile<true, true, Epi><<<grid, kThreads, smem, st>>>(a, epi);
    } else {
        const size_t smem = (size_t)a.prefix * sizeof(float);
        if (p.pattern) tc_spmv_tile<false, false, Epi><<<grid, kThreads, smem, st>>>(a, epi);
        else tc_spmv_tile<false, true, Epi><<<grid, kThreads, smem, st>>>(a, epi);
    }
    return cudaGetLastError();
}

// Launch every non-empty tile of `p` in ascending order.
template <class Epi>
cudaError_t launch_tiles(const spmv_plan_s& p, const std::vector<int>& grids, const float* xp,
                         const Epi& epi, cudaStream_t st) {
    for (int32_t t = 0; t <= p.num_tiles; ++t) {
        if (p.tiles[t].wl_end == p.tiles[t].wl_begin) continue;
        cudaError_t e = launch_tile(p, t, grids[t], xp, epi, st);
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
    int nb = 0;
    if ((e = cudaFuncSetAttribute(kgl, cudaFuncAttributeMaxDynamicSharedMemorySize, max_dyn))) return e;
    // unstaged tiles gather x through L1: ask for the largest L1 (smallest shared carve-out)
    if (p.x_prefix == 0 && p.l1_carveout >= 0 &&
        (e = cudaFuncSetAttribute(kgl, cudaFuncAttributePreferredSharedMemoryCarveout, p.l1_carveout))) return e;
    if (p.x_prefix * 4 > max_dyn) p.x_prefix = max_dyn / 4;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kgl, kThreads, (size_t)p.x_prefix * 4))) return e;
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
    if (p.stream) {  // classic attributes above stay set: tiles that do not fit fall back
        int optin = 0;
        if ((e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, p.device))) return e;
        auto k0 = p.pattern ? tc_spmv_wstream<true, false, Epi> : tc_spmv_wstream<true, true, Epi>;
        auto k1 = p.pattern ? tc_spmv_wstream<false, false, Epi> : tc_spmv_wstream<false, true, Epi>;
        cudaFuncAttributes fa0, fa1;
        if ((e = cudaFuncGetAttributes(&fa0, k0)) || (e = cudaFuncGetAttributes(&fa1, k1))) return e;
        const int dyn = optin - (int)std::max(fa0.sharedSizeBytes, fa1.sharedSizeBytes);
        if ((e = cudaFuncSetAttribute(k0, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn)) ||
            (e = cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn))) return e;
        p.max_dyn_smem = std::min(p.max_dyn_smem > 0 ? p.max_dyn_smem : dyn, dyn);
        grids.assign(p.num_tiles + 1, p.stream_grid);
    }
    return cudaSuccess;
}

}  // namespace tc
