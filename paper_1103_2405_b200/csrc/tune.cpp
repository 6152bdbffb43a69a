// tune.cpp -- the paper's auto-tuner and performance model (Sec. 3.3, Appendix E), on B200.
//
//   offline table   Performance(w, h): whole-GPU slots/s when every warp runs a w x h workload
//                   (reading R20), measured by bench/calibrate.py for x cached
//                   (staged in shared memory: dense tiles) and uncached (L1/L2 gathers: the
//                   remainder, L160), per workload kind and value type
//   PM(T, WL)       Alg. 3 (L382-L407, Eq. 1-5): walk the tile's packing with workload size WL,
//                   group workloads into waves of MAX_ACT_WARP warps, t_i = Size_i / P_i with
//                   P_i the mean table throughput of the wave, total = sum t_i
//   Partition(T)    Alg. 2 (L358-L375): argmin of PM over the candidate WLs (strict <)
//   tile count      Alg. 1 (L335-L356): tiles while the first column has >= 2 entries (the
//                   upper bound), then the count with the least predicted total (B200 model)
// B200 additions: rows longer than WL are split (R21), so WL candidates
// are powers of two; each tile launch also pays a launch gap, the staging of its x segment
// (dense tiles) and the read-modify-write of y for rows an earlier tile touched.
#include "tune.h"

#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <sstream>
#include <string>

#include "plan_impl.h"

namespace tc {

static constexpr int32_t kDefaultTileWidth = 24576;
static constexpr int32_t kDefaultWL = 1024;

// ------------------------------------------------------------------ offline table
struct PerfTable {
    // key: (x mode, valued, kind) -> grid over (log2 w, log2 h); x mode 0 = uncached with uniform
    // columns (a remainder whose hub columns went to dense tiles), 1 = cached (x segment in
    // shared memory), 2 = uncached with power-law columns (single-tile plans: hubs hit L1)
    struct Grid { std::vector<double> lw, lh; std::vector<std::vector<double>> v; };
    std::map<int, Grid> grids;
    double launch_us = 3.0;         // per tile launch gap
    double stage_GBps = 6000.0;     // chip-wide L2 -> shared memory staging bandwidth
    double rmw_GBps = 4000.0;       // y read-modify-write of accumulating rows
    double tail_frac = 0.0;         // launch tail: this fraction of one workload's duration under load
    double l2_budget_bytes = 96e6;  // x spans above this are served by DRAM (mode 3, reading R32)
    // two-phase tiles: measured time per work item of one persistent CTA
    double pb_item_us = 3.2;           // valued
    double pb_item_us_pattern = 2.95;
    double pb_launch_us = 4.0;
    int max_act_warp = 148 * 32;
    bool loaded = false;
    std::string source = "built-in";

    static int key(int mode, bool valued, int kind) { return mode * 4 + (valued ? 2 : 0) + (kind == KIND_CM ? 1 : 0); }

    // bilinear interpolation in (log2 w, log2 h), clamped to the measured range
    double lookup(int mode, bool valued, int kind, double w, double h) const {
        auto it = grids.find(key(mode, valued, kind));
        if (it == grids.end() && (mode == 2 || mode == 3)) it = grids.find(key(0, valued, kind));
        const bool cached = mode == 1;
        if (it == grids.end() || it->second.lw.empty() || it->second.lh.empty()) return analytic(cached, valued, kind, w, h);
        const Grid& g = it->second;
        auto locate = [](const std::vector<double>& ax, double v, int& i, double& f) {
            if (v <= ax.front()) { i = 0; f = 0; return; }
            if (v >= ax.back()) { i = (int)ax.size() - 1; f = 0; return; }
            i = (int)(std::upper_bound(ax.begin(), ax.end(), v) - ax.begin()) - 1;
            f = (v - ax[i]) / (ax[i + 1] - ax[i]);
        };
        int i, j; double fi, fj;
        locate(g.lw, std::log2(std::max(w, 1.0)), i, fi);
        locate(g.lh, std::log2(std::max(h, 1.0)), j, fj);
        auto at = [&](int a, int b) {
            a = std::min(a, (int)g.lw.size() - 1); b = std::min(b, (int)g.lh.size() - 1);
            return g.v[a][b];
        };
        double v00 = at(i, j), v10 = at(i + 1, j), v01 = at(i, j + 1), v11 = at(i + 1, j + 1);
        if (fi == 0) { v10 = v00; v11 = v01; }
        if (fj == 0) { v01 = v00; v11 = v10; }
        double v = (1 - fi) * (1 - fj) * v00 + fi * (1 - fj) * v10 + (1 - fi) * fj * v01 + fi * fj * v11;
        return v > 0 ? v : analytic(cached, valued, kind, w, h);
    }
    // used only when no measured table is available: slots/s bounded by HBM streaming and by
    // the gather rate (shared memory ~1.3 T/s, L1/L2 ~0.27 T/s)
    static double analytic(bool cached, bool valued, int kind, double w, double h) {
        const double bytes = valued ? 8.0 : 4.0;
        const double hbm = 6.4e12 / bytes;
        const double gather = cached ? 1.3e12 : 2.7e11;
        double eff = 1.0;
        if (kind == KIND_RM) eff = std::min(1.0, w / 128.0 + 0.25);
        else eff = std::min(1.0, 0.5 + w / 32.0);
        (void)h;
        return eff * std::min(hbm, gather);
    }
};

static bool parse_table(const std::string& text, PerfTable& T) {
    // minimal reader for the calibration file: "key": number and "entries": [[c,v,k,w,h,s],...]
    auto num_after = [&](const char* k, double& out) {
        size_t p = text.find(std::string("\"") + k + "\"");
        if (p == std::string::npos) return false;
        p = text.find(':', p);
        if (p == std::string::npos) return false;
        out = std::strtod(text.c_str() + p + 1, nullptr);
        return true;
    };
    double v;
    if (num_after("launch_us", v)) T.launch_us = v;
    if (num_after("stage_GBps", v)) T.stage_GBps = v;
    if (num_after("rmw_GBps", v)) T.rmw_GBps = v;
    if (num_after("tail_frac", v)) T.tail_frac = v;
    if (num_after("max_act_warp", v)) T.max_act_warp = (int)v;
    if (num_after("l2_budget_bytes", v)) T.l2_budget_bytes = v;
    if (num_after("pb_item_us", v)) T.pb_item_us = v;
    if (num_after("pb_item_us_pattern", v)) T.pb_item_us_pattern = v;
    if (num_after("pb_launch_us", v)) T.pb_launch_us = v;
    size_t p = text.find("\"entries\"");
    if (p == std::string::npos) return false;
    p = text.find('[', p);
    if (p == std::string::npos) return false;
    std::map<int, std::map<std::pair<double, double>, double>> raw;
    const char* s = text.c_str() + p + 1;
    int n = 0;
    while (*s) {
        while (*s && *s != '[' && *s != ']') ++s;
        if (!*s || *s == ']') break;
        ++s;
        double f[6];
        int k = 0;
        while (k < 6 && *s && *s != ']') {
            while (*s == ' ' || *s == ',' || *s == '\n') ++s;
            char* e = nullptr;
            f[k] = std::strtod(s, &e);
            if (e == s) return false;
            s = e;
            ++k;
        }
        while (*s && *s != ']') ++s;
        if (*s) ++s;
        if (k != 6) return false;
        raw[PerfTable::key((int)f[0], f[1] != 0, (int)f[2])][{std::log2(f[3]), std::log2(f[4])}] = f[5];
        ++n;
    }
    for (auto& kv : raw) {
        PerfTable::Grid g;
        for (auto& e : kv.second) { g.lw.push_back(e.first.first); g.lh.push_back(e.first.second); }
        std::sort(g.lw.begin(), g.lw.end()); g.lw.erase(std::unique(g.lw.begin(), g.lw.end()), g.lw.end());
        std::sort(g.lh.begin(), g.lh.end()); g.lh.erase(std::unique(g.lh.begin(), g.lh.end()), g.lh.end());
        g.v.assign(g.lw.size(), std::vector<double>(g.lh.size(), 0.0));
        // fill: nearest measured neighbour in h for holes (rm shapes need w >= h)
        for (size_t i = 0; i < g.lw.size(); ++i)
            for (size_t j = 0; j < g.lh.size(); ++j) {
                double best = 0, bd = 1e30;
                for (auto& e : kv.second) {
                    double d = std::fabs(e.first.first - g.lw[i]) * 4 + std::fabs(e.first.second - g.lh[j]);
                    if (d < bd) { bd = d; best = e.second; }
                }
                g.v[i][j] = best;
            }
        T.grids[kv.first] = g;
    }
    return n > 0;
}

static const PerfTable& table_for(const char* path_opt) {
    static PerfTable builtin;
    static std::map<std::string, PerfTable> cache;
    std::string path = path_opt ? path_opt : "";
    if (path.empty()) {
        const char* env = std::getenv("TCSPMV_PERF_TABLE");
        if (env) path = env;
    }
    if (path.empty()) {
        Dl_info info;
        if (dladdr((void*)&table_for, &info) && info.dli_fname) {
            std::string so = info.dli_fname;
            size_t k = so.rfind('/');
            std::string dir = k == std::string::npos ? "." : so.substr(0, k);
            path = dir + "/../data/perf_table_b200.json";
        }
    }
    auto it = cache.find(path);
    if (it != cache.end()) return it->second;
    std::ifstream f(path);
    if (!f) return builtin;
    std::stringstream ss;
    ss << f.rdbuf();
    PerfTable T;
    if (!parse_table(ss.str(), T)) return builtin;
    T.loaded = true;
    T.source = path;
    return cache.emplace(path, T).first->second;
}

double stream_pass_us(const spmv_options& opt, double bytes) {
    const PerfTable& T = table_for(opt.perf_table_path);
    return T.launch_us + bytes / (T.stage_GBps * 1e3);
}

// ------------------------------------------------------------------ Alg. 3 on the packing walk
// hist: (length, count) pairs, lengths descending (a tile's ranked rows).  Walks the same packing
// rules as pack_layout and charges every workload to its wave.
static double pm_tile(const std::vector<std::pair<int64_t, int64_t>>& hist, int64_t WL, int align,
                      bool split, int ell_h, int cached, bool valued, const PerfTable& T,
                      int64_t* n_workloads = nullptr, int32_t orient = 0) {
    const int64_t M = std::max(1, T.max_act_warp);      // MAX_ACT_WARP (Eq. 1)
    double total = 0.0, P = 0.0, S = 0.0, P_all = 0.0;
    int64_t cnt = 0, nw = 0;
    auto add = [&](int kind, int64_t w, int64_t h, int64_t slots) {   // Alg. 3 lines 11-14
        const double perf = T.lookup(cached, valued, kind, (double)std::max<int64_t>(w, 1), (double)h);
        P += perf;
        P_all += perf;
        S += (double)slots;
        ++cnt; ++nw;
        if (cnt == M) { total += S / (P / (double)cnt); P = S = 0.0; cnt = 0; }   // Eq. 3-5
    };
    auto rup = [](int64_t a, int64_t b) { return (a + b - 1) / b * b; };
    // cursor over the ranked rows, stored as (length, count) groups
    size_t g = 0;
    int64_t off = 0, remaining = 0;
    for (auto& h : hist) remaining += h.second;
    auto advance = [&](int64_t k) {
        remaining -= k;
        while (k > 0 && g < hist.size()) {
            const int64_t c = std::min(k, hist[g].second - off);
            off += c; k -= c;
            if (off == hist[g].second) { ++g; off = 0; }
        }
    };
    while (remaining > 0) {                                  // Alg. 3 lines 7-16 (packing walk)
        const int64_t w = hist[g].first;
        const int64_t hq = std::max<int64_t>(1, WL / std::max<int64_t>(w, 1));
        if (orient == 3 && !(split && w > WL)) {
            // TILE-COO workload: whole rows while at most WL entries (at least one), padded to 32
            // slots; charged at the row-major table shape (w = slots, h = 1)
            int64_t tot = 0, h = 0, oo = off;
            size_t gg = g;
            while (gg < hist.size()) {
                const int64_t L = hist[gg].first, avail = hist[gg].second - oo;
                int64_t k = L > 0 ? std::min<int64_t>(avail, (WL - tot) / L) : avail;
                if (h == 0 && k == 0) k = 1;
                if (k <= 0) break;
                tot += k * L; h += k; oo += k;
                if (oo < hist[gg].second) break;
                ++gg; oo = 0;
                if (gg < hist.size() && split && hist[gg].first > WL) break;
            }
            const int64_t wp = rup(tot, 32);
            add(KIND_RM, wp, 1, wp);
            advance(h);
            continue;
        }
        if (split && w > WL) {                               // R21: one-row chunks
            for (int64_t c = 0; c * WL < w; ++c) {
                const int64_t part = std::min<int64_t>(WL, w - c * WL), wp = rup(part, align);
                add(KIND_RM, wp, 1, wp);
            }
            advance(1);
        } else if (row_major(orient == 3 ? 0 : orient, w, hq)) {   // row major
            const int64_t h = std::min<int64_t>(hq, remaining), wp = rup(w, align);
            add(KIND_RM, wp, h, h * wp);
            advance(h);
        } else {                                             // column major
            const int64_t take = std::min<int64_t>(rup(hq, ell_h), remaining);
            const int64_t hs = rup(take, ell_h);
            add(KIND_CM, w, hs, hs * w);
            advance(take);
        }
    }
    if (cnt > 0) total += S / (P / (double)cnt);             // last (partial) wave, R23
    // B200 term (reading R31): the launch ends when its last workload does; on average the
    // stragglers add tail_frac of one workload's duration under load, WL / (mean P / MAX_ACT_WARP)
    if (nw > 0 && T.tail_frac > 0.0) total += T.tail_frac * (double)WL * (double)M / (P_all / (double)nw);
    if (n_workloads) *n_workloads = nw;
    return total;   // seconds
}

// Alg. 2 in B200 mode: candidates are powers of two (rows longer than WL split) plus the paper's
// multiples of the longest row; paper mode (no split) keeps WL >= the longest row.
static void partition_tile(const std::vector<std::pair<int64_t, int64_t>>& hist, const BuildParams& bp,
                           int cached, bool valued, const PerfTable& T, int32_t& opt_wl, double& opt_t) {
    const int64_t L = hist.empty() ? 1 : std::max<int64_t>(1, hist[0].first);
    int64_t nnz = 0;
    for (auto& h : hist) nnz += h.first * h.second;
    std::vector<int64_t> cand;
    if (bp.split) {
        // reading R21: rows longer than WL are split, so WL is free: powers of two from one warp's
        // slots up, and the paper's multiples of the longest row, up to max(WL_low, 32768) (the
        // paper's table bound)
        const int64_t up = std::max<int64_t>(L, 32768);
        for (int64_t c = 32; c <= up; c *= 2) cand.push_back(c);
        int nm = 0;
        for (int64_t c = L; c <= up && nm < 96; c += L, ++nm) cand.push_back(c);
        std::sort(cand.begin(), cand.end());
        cand.erase(std::unique(cand.begin(), cand.end()), cand.end());
    } else {
        const int64_t up = std::max<int64_t>(L, nnz / std::max(1, T.max_act_warp));
        for (int64_t c = L; c <= up && cand.size() < 64; c += L) cand.push_back(c);
        if (cand.empty()) cand.push_back(L);
    }
    // the candidates are independent model walks: evaluated in parallel, reduced in candidate
    // order (strict <, so the smallest WL wins ties, R22)
    std::vector<double> tt(cand.size());
    #pragma omp parallel for schedule(dynamic, 1)
    for (int64_t i = 0; i < (int64_t)cand.size(); ++i)
        tt[i] = pm_tile(hist, cand[i], bp.align_rm, bp.split, bp.ell_h, cached, valued, T, nullptr, bp.orient);
    opt_t = INFINITY; opt_wl = (int32_t)cand[0];
    for (size_t i = 0; i < cand.size(); ++i)
        if (tt[i] < opt_t) { opt_t = tt[i]; opt_wl = (int32_t)cand[i]; }
}

struct Choice { int32_t tw, T; std::vector<int32_t> wl; std::vector<double> us; double total; };

// x regime of tile t (the offline table's x mode): 1 = staged in shared memory; otherwise 3 when
// the tile's x span exceeds the L2 budget (gathers from DRAM, reading R32), 2 when the tile holds
// the hub columns (single tile or unstaged first tile: hubs hit L1), else 0
static int x_mode(const Prepared& P, int32_t tw, int32_t T, int32_t t, bool cached, const PerfTable& tab) {
    if (cached) return 1;
    const int64_t lo = std::min<int64_t>((int64_t)t * tw, P.n_cols);
    const int64_t hi = t < T ? std::min<int64_t>((int64_t)(t + 1) * tw, P.n_cols) : P.n_cols;
    if ((double)(hi - lo) * 4.0 > tab.l2_budget_bytes) return 3;
    return t == 0 ? 2 : 0;
}

static Choice evaluate(const Prepared& P, const spmv_options& opt, const BuildParams& base, int32_t tw,
                       int32_t T, const PerfTable& tab, bool stage,
                       const std::vector<std::vector<std::pair<int64_t, int64_t>>>& hist) {
    Choice c{tw, T, {}, {}, 0.0};
    const bool valued = !P.pattern;
    for (int32_t t = 0; t <= T; ++t) {
        const bool cached = stage && t < T && opt.stage_x != 0;
        const int mode = x_mode(P, tw, T, t, cached, tab);
        int32_t wl = kDefaultWL;
        double sec = 0.0;
        if (opt.workload_sizes) wl = opt.workload_sizes[std::min(t, opt.num_tiles >= 0 ? opt.num_tiles : t)];
        else if (opt.workload_size > 0) wl = opt.workload_size;
        BuildParams bt = base;                  // TILE-COO: COO dense tiles, composite remainder
        if (bt.orient == 3 && t == T) bt.orient = 0;
        if (opt.workload_sizes || opt.workload_size > 0) {
            sec = pm_tile(hist[t], wl, bt.align_rm, bt.split, bt.ell_h, mode, valued, tab, nullptr, bt.orient);
        } else {
            partition_tile(hist[t], bt, mode, valued, tab, wl, sec);
        }
        int64_t rows = 0, nnz = 0;
        for (auto& h : hist[t]) { rows += h.second; nnz += h.first * h.second; }
        double us = sec * 1e6;
        if (rows > 0) {
            us += tab.launch_us;
            if (cached) us += (double)tw * 4.0 * 148 / (tab.stage_GBps * 1e3);
            if (t > 0) us += (double)rows * 8.0 / (tab.rmw_GBps * 1e3);   // y partial read + write
        }
        c.wl.push_back(wl);
        c.us.push_back(us);
        c.total += us;
    }
    return c;
}

spmv_status choose_params(const Prepared& P, const spmv_options& opt, int sm_count,
                          BuildParams& bp, std::vector<double>& pred_us, int32_t* table_loaded) {
    if (opt.orient == -1) {
        // CSR-vector (row major only) and ELL (column major only) are special cases of the
        // tile-composite model; "the best predicted kernel can be chosen" -- evaluate them, the
        // composite and TILE-COO
        double best = INFINITY;
        for (int32_t o : {0, 1, 2, 3}) {
            spmv_options oo = opt;
            oo.orient = o;
            BuildParams b;
            std::vector<double> pr;
            spmv_status st = choose_params(P, oo, sm_count, b, pr, table_loaded);
            if (st) return st;
            double tot = 0.0;
            for (double u : pr) tot += u;
            if (tot < best) { best = tot; bp = b; pred_us = pr; }
        }
        return SPMV_OK;
    }
    bp.align_rm = opt.align_rm;
    bp.split = opt.split_long_rows != 0;
    bp.camping = opt.camping_pad != 0;
    bp.ell_h = opt.ell_h;
    bp.orient = opt.orient;
    PerfTable tab = table_for(opt.perf_table_path);
    tab.max_act_warp = std::max(1, (int)((int64_t)tab.max_act_warp * sm_count / 148));
    if (opt.perf_table_path && !tab.loaded) { set_error("performance table unreadable"); return SPMV_ETABLE; }
    if (table_loaded) *table_loaded = tab.loaded ? 1 : 0;

    std::vector<int32_t> tws;
    if (opt.tile_width > 0) tws.push_back(opt.tile_width);
    else tws = {12288, 24576, 49152};
    Choice best{0, 0, {}, {}, INFINITY};
    for (int32_t tw : tws) {
        const int64_t max_tiles = P.n_cols > 0 ? (P.n_cols + tw - 1) / tw : 0;
        std::vector<int32_t> Ts;
        if (opt.num_tiles >= 0) Ts.push_back((int32_t)std::min<int64_t>(opt.num_tiles, max_tiles));
        else {
            // Alg. 1 gives the upper bound; the model picks the count (B200 terms included).
            // Columns in the caller's order (keep_col_order) are not length-sorted: no dense
            // tiles, only the L2-sized ones below
            const int32_t Tp = opt.keep_col_order ? 0 : std::min<int32_t>(paper_tile_count(P, tw), 16);
            for (int32_t T = 0; T <= Tp; T = (T < 4 ? T + 1 : T * 2)) Ts.push_back(T);
            if (Ts.back() != Tp) Ts.push_back(Tp);
        }
        Ts.erase(std::remove_if(Ts.begin(), Ts.end(), [](int32_t T) { return T > 63; }), Ts.end());
        std::vector<std::vector<std::vector<std::pair<int64_t, int64_t>>>> hists;
        tile_histograms_multi(P, tw, Ts, hists);           // one pass over the entries per width
        for (size_t j = 0; j < Ts.size(); ++j) {
            Choice c = evaluate(P, opt, bp, tw, Ts[j], tab, true, hists[j]);
            if (c.total < best.total) best = c;
        }
        if (opt.num_tiles >= 0 && opt.tile_width > 0) break;
    }
    // x beyond L2 (c4-sized graphs): also L2-sized unstaged tiles, the paper's Solution 1 one
    // level up (the tile's x segment stays in L2 instead of shared memory)
    if (opt.tile_width <= 0 && (double)P.n_cols * 4.0 > tab.l2_budget_bytes) {
        for (int32_t tw : {1 << 20, 1 << 21, 1 << 22, 1 << 23}) {
            if ((double)tw * 4.0 > tab.l2_budget_bytes) continue;
            const int64_t max_tiles = (P.n_cols + tw - 1) / tw;
            std::vector<int32_t> Ts;
            for (int32_t T : {1, 2, 4})   // 6 / 8 / 12 measured equal on c4 (profiles/r01_c4_model.jsonl)
                if ((opt.num_tiles < 0 || T == opt.num_tiles) && T < max_tiles) Ts.push_back(T);
            if (Ts.empty()) continue;
            std::vector<std::vector<std::vector<std::pair<int64_t, int64_t>>>> hists;
            tile_histograms_multi(P, tw, Ts, hists);
            for (size_t j = 0; j < Ts.size(); ++j) {
                Choice c = evaluate(P, opt, bp, tw, Ts[j], tab, false, hists[j]);
                if (c.total < best.total) best = c;
            }
        }
    }
    if (best.wl.empty()) { set_error("no tiling candidate"); return SPMV_EINVAL; }
    bp.tile_width = best.tw;
    bp.num_tiles = best.T;
    bp.wl = best.wl;
    pred_us = best.us;
    return SPMV_OK;
}

void predict_plan(spmv_plan_s& p, const std::vector<double>& pred_us) {
    p.predicted_us = 0.0;
    for (size_t t = 0; t < p.tiles.size() && t < pred_us.size(); ++t) {
        p.tiles[t].pred_us = pred_us[t];
        p.predicted_us += pred_us[t];
    }
}

// ------------------------------------------------------------------ two-phase tiles (pb.h)
// Group size: the live part of the partial buffer (about four groups: one being expanded, one
// being reduced, the ones in between) stays in L2 beside x, capped at 8 M products (a larger group
// holds more bins than a chunk's run table, so its chunks shrink; measured on c2 and c4,
// DESIGN.md 7c).
PbParams pb_params(const spmv_options& opt, int64_t n_cols, int64_t nnz) {
    PbParams prm;
    const PerfTable tab = table_for(opt.perf_table_path);
    if (opt.pb_region > 0) prm.rcap = opt.pb_region;
    if (opt.pb_chunk > 0) prm.ccap = opt.pb_chunk;
    if (opt.pb_xcap > 0) prm.xcap = opt.pb_xcap;
    prm.pcap = std::min<int32_t>(65535, std::max<int32_t>(1024, prm.rcap + prm.rcap / 2));
    if (opt.pb_group > 0) prm.gcap = opt.pb_group;
    else {
        const double free_l2 = std::max(0.0, tab.l2_budget_bytes - 4.0 * (double)n_cols);
        prm.gcap = std::min<int64_t>(8 << 20, std::max<int64_t>(1 << 20, (int64_t)(free_l2 / (4.0 * 4.0))));
    }
    (void)nnz;
    return prm;
}

// Model of the two-phase tiles.  Both phases run out of shared-memory stages filled by bulk
// copies, so time is set by how many items the persistent CTAs get through: t = items * t_item /
// CTAs + launch, with t_item measured on B200 (a CTA's two-stage pipeline at two CTAs per SM;
// defaults 3.2 / 2.95 us valued / pattern from round-2's first layout (c2 29.7 K items in 325 us);
// the shipped table carries 3.32 / 3.15 us, refitted to the x segment cap of 6144: c2 28.6 K items
// in 325 / 309 us).
// The item count is estimated from the parameters: bins of ~rcap products, and chunks cut by
// whichever of ccap entries, xcap columns or nrcap distinct bins binds first.
double pb_predict_us(const spmv_options& opt, int64_t n_rows, int64_t n_cols, int64_t nnz, bool valued,
                     const PbParams& prm) {
    const PerfTable tab = table_for(opt.perf_table_path);
    const double m = (double)nnz;
    if (m <= 0) return tab.pb_launch_us;
    const double groups = std::max(1.0, std::ceil(m / (double)prm.gcap));
    const double bins = std::max(m / (0.8 * prm.rcap), (double)n_rows / prm.maxrows);
    const double per_col = m / (groups * std::max<double>(1.0, (double)n_cols));   // entries per column per group
    const double bins_g = bins / groups;
    double e_chunk = std::min<double>(prm.ccap, std::max(1.0, prm.xcap * per_col));
    if (bins_g > 2.0 * prm.nrcap) e_chunk = std::min<double>(e_chunk, prm.nrcap);
    const double chunks = m / e_chunk;
    const double ctas = 2.0 * 148.0;
    return tab.pb_launch_us + (chunks + bins) * (valued ? tab.pb_item_us : tab.pb_item_us_pattern) / ctas;
}

// the same model over a built layout's actual item count
double pb_predict_items_us(const spmv_options& opt, int64_t items, bool valued) {
    const PerfTable tab = table_for(opt.perf_table_path);
    return tab.pb_launch_us + (double)items * (valued ? tab.pb_item_us : tab.pb_item_us_pattern) / (2.0 * 148.0);
}

}  // namespace tc
