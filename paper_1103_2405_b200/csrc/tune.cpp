// tune.cpp -- parameter choice.  Explicit options are honoured as given; "auto" values are
// chosen here (the performance-model auto-tuner replaces the defaults).
#include "tune.h"

#include <algorithm>

#include "plan_impl.h"

namespace tc {

static constexpr int32_t kDefaultTileWidth = 24576;   // 96 KB of x per CTA: 2 CTAs per SM
static constexpr int32_t kDefaultWL = 1024;

spmv_status choose_params(const Prepared& P, const spmv_options& opt, int sm_count,
                          BuildParams& bp, std::vector<double>& pred_us) {
    (void)sm_count;
    bp.align_rm = opt.align_rm;
    bp.split = opt.split_long_rows != 0;
    bp.camping = opt.camping_pad != 0;
    bp.ell_h = opt.ell_h;
    bp.tile_width = opt.tile_width > 0 ? opt.tile_width : kDefaultTileWidth;
    const int64_t max_tiles = P.n_cols > 0 ? (P.n_cols + bp.tile_width - 1) / bp.tile_width : 0;
    if (opt.num_tiles >= 0) {
        // explicit counts are clipped to the tiles that exist (ceil(n_cols / tile_width))
        bp.num_tiles = (int32_t)std::min<int64_t>(opt.num_tiles, max_tiles);
    } else {
        bp.num_tiles = std::min<int32_t>(paper_tile_count(P, bp.tile_width), 2);
    }
    if (bp.num_tiles > 63) { set_error("more than 63 dense tiles"); return SPMV_ERANGE; }
    const int32_t T = bp.num_tiles;
    bp.wl.assign(T + 1, kDefaultWL);
    if (opt.workload_sizes) {
        // num_tiles + 1 values as given; after clipping the remainder keeps the last value
        for (int32_t t = 0; t < T; ++t) bp.wl[t] = opt.workload_sizes[t];
        bp.wl[T] = opt.workload_sizes[opt.num_tiles >= 0 ? opt.num_tiles : T];
    } else if (opt.workload_size > 0) {
        std::fill(bp.wl.begin(), bp.wl.end(), opt.workload_size);
    } else if (!bp.split) {
        // paper lower bound (Alg. 2 line 3): WL >= the tile's longest row
        std::vector<std::vector<std::pair<int64_t, int64_t>>> hist;
        tile_histograms(P, bp.tile_width, T, hist);
        for (int32_t t = 0; t <= T; ++t) {
            int64_t L = hist[t].empty() ? 1 : std::max<int64_t>(1, hist[t][0].first);
            bp.wl[t] = (int32_t)std::max<int64_t>(kDefaultWL, L);
        }
    }
    pred_us.assign(T + 1, 0.0);
    return SPMV_OK;
}

void predict_plan(spmv_plan_s& p, const std::vector<double>& pred_us) {
    p.predicted_us = 0.0;
    for (size_t t = 0; t < p.tiles.size() && t < pred_us.size(); ++t) {
        p.tiles[t].pred_us = pred_us[t];
        p.predicted_us += pred_us[t];
    }
}

}  // namespace tc
