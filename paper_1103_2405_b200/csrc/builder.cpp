// builder.cpp -- host-side format builder (steps a1-a5 of SURVEY.md 8(a); Format v1).
//
//   a1/a2  column lengths; columns relabelled by (length desc, id asc) with a counting sort
//          (Solution 2; "sorted by counting sort in linear time", L98)
//   a3     dense tiles of tile_width relabelled columns + one remainder tile (Solution 1, L56-L60;
//          remainder "as one matrix tile", L90-L92)
//   a4     rows of each tile ranked by in-tile length, high to low (Observation 5 / Solution 3, L86-L88)
//   a5     workload packing per Alg. 3 lines 8-15 (L392-L401): w = first row length, h = WL / w;
//          w >= h -> row major (CSR-vector), else column major (ELL); rows padded to w; w padded
//          to align_rm (row major) or h to ell_h (column major) (Solution 3, L88, L94); optional
//          partition-camping pad (L96); rows longer than WL split into chunks (B200, reading R21).
#include <algorithm>
#include <atomic>
#include <cstring>
#include <numeric>

#include "plan.h"

namespace tc {

static inline int64_t roundup(int64_t a, int64_t b) { return ((a + b - 1) / b) * b; }

spmv_status prepare(int64_t n_rows, int64_t n_cols, int64_t nnz, const int64_t* row_ptr,
                    const int32_t* col, const float* val, bool pattern, Prepared& P, bool keep_order) {
    if (n_rows < 0 || n_cols < 0 || nnz < 0) { set_error("negative size"); return SPMV_EINVAL; }
    if (n_rows >= (int64_t(1) << 29)) { set_error("n_rows must be < 2^29"); return SPMV_ERANGE; }
    if (n_cols > INT32_MAX - 1) { set_error("n_cols must be < 2^31-1"); return SPMV_ERANGE; }
    if (!row_ptr || (nnz > 0 && !col) || (nnz > 0 && !pattern && !val)) {
        set_error("null input pointer"); return SPMV_EINVAL;
    }
    if (row_ptr[0] != 0 || row_ptr[n_rows] != nnz) { set_error("row_ptr[0] != 0 or row_ptr[n] != nnz"); return SPMV_EINVAL; }
    std::atomic<int> bad{0};
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n_rows; ++i)
        if (row_ptr[i + 1] < row_ptr[i]) bad = 1;
    if (bad) { set_error("row_ptr not monotone"); return SPMV_EINVAL; }
    #pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < nnz; ++k)
        if (col[k] < 0 || col[k] >= n_cols) bad = 2;
    if (bad) { set_error("column index out of range"); return SPMV_EINVAL; }

    P.n_rows = n_rows; P.n_cols = n_cols; P.nnz = nnz; P.pattern = pattern;
    // a1: column lengths
    std::vector<int64_t> len(n_cols, 0);
    #pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < nnz; ++k) __atomic_fetch_add(&len[col[k]], 1, __ATOMIC_RELAXED);
    // a2: counting sort by (length desc, id asc)
    int64_t maxlen = 0;
    for (int64_t j = 0; j < n_cols; ++j) maxlen = std::max(maxlen, len[j]);
    std::vector<int64_t> start(maxlen + 2, 0);
    for (int64_t j = 0; j < n_cols; ++j) start[maxlen - len[j] + 1]++;   // bucket b = maxlen - len
    for (int64_t b = 0; b <= maxlen; ++b) start[b + 1] += start[b];
    P.perm.assign(n_cols, 0);
    P.inv.assign(n_cols, 0);
    for (int64_t j = 0; j < n_cols; ++j) {
        // keep_order: the caller's column order is kept (its x is laid out by someone else)
        int64_t pos = keep_order ? j : start[maxlen - len[j]]++;
        P.perm[pos] = (int32_t)j;
        P.inv[j] = (int32_t)pos;
    }
    P.collen.assign(n_cols, 0);
    for (int64_t k = 0; k < n_cols; ++k) P.collen[k] = len[P.perm[k]];
    // relabelled rows, entries ordered by (relabelled column, original position)
    P.rp.assign(row_ptr, row_ptr + n_rows + 1);
    P.kcol.resize(nnz);
    if (!pattern) P.kval.resize(nnz);
    int64_t mrl = 0;
    #pragma omp parallel reduction(max : mrl)
    {
        std::vector<uint64_t> key;
        #pragma omp for schedule(dynamic, 256)
        for (int64_t i = 0; i < n_rows; ++i) {
            int64_t s = row_ptr[i], e = row_ptr[i + 1], L = e - s;
            mrl = std::max(mrl, L);
            if (L == 0) continue;
            key.resize(L);
            for (int64_t p = 0; p < L; ++p) key[p] = ((uint64_t)(uint32_t)P.inv[col[s + p]] << 32) | (uint64_t)p;
            std::sort(key.begin(), key.end());
            for (int64_t p = 0; p < L; ++p) {
                int64_t src = s + (int64_t)(key[p] & 0xFFFFFFFFu);
                P.kcol[s + p] = (int32_t)(key[p] >> 32);
                if (!pattern) P.kval[s + p] = val[src];
            }
        }
    }
    P.max_row_len = mrl;
    return SPMV_OK;
}

// Alg. 1 lines 4-8, reading R10: continue while NTile * TW < n.
int32_t paper_tile_count(const Prepared& P, int64_t tw) {
    int32_t t = 0;
    while ((int64_t)t * tw < P.n_cols) {
        if (P.collen[(int64_t)t * tw] <= 1) break;
        ++t;
    }
    return t;
}

static inline int32_t tile_of(int64_t k, int64_t tw, int32_t T) {
    int64_t t = k / tw;
    return t < T ? (int32_t)t : T;
}

// Row-length histograms of every tile for several tile counts at one tile width, in one pass over
// the entries (the auto-tuner evaluates all candidate counts of a width).  Thread-local dense
// counters for lengths below kSmall, atomics only for the rare longer segments.
void tile_histograms_multi(const Prepared& P, int64_t tw, const std::vector<int32_t>& Ts,
                           std::vector<std::vector<std::vector<std::pair<int64_t, int64_t>>>>& out) {
    constexpr int64_t kSmall = 4096;
    const size_t J = Ts.size();
    int32_t Tmax = 0;
    for (int32_t T : Ts) Tmax = std::max(Tmax, T);
    std::vector<size_t> base(J + 1, 0);                     // flat (j, t) slot index
    for (size_t j = 0; j < J; ++j) base[j + 1] = base[j] + (size_t)Ts[j] + 1;
    const size_t S = base[J];
    const int64_t cap = P.max_row_len + 1;
    std::vector<std::vector<int64_t>> big(S, std::vector<int64_t>(cap > kSmall ? cap : 0, 0));
    std::vector<int64_t> small(S * kSmall, 0);
    #pragma omp parallel
    {
        std::vector<int64_t> loc(S * kSmall, 0);
        std::vector<int64_t> seg(Tmax + 1);
        auto add = [&](size_t slot, int64_t len) {
            if (len < kSmall) loc[slot * kSmall + len]++;
            else __atomic_fetch_add(&big[slot][len], 1, __ATOMIC_RELAXED);
        };
        #pragma omp for schedule(dynamic, 4096)
        for (int64_t i = 0; i < P.n_rows; ++i) {
            const int64_t s = P.rp[i], e = P.rp[i + 1];
            if (s == e) { for (size_t j = 0; j < J; ++j) add(base[j] + Ts[j], 0); continue; }
            std::fill(seg.begin(), seg.end(), 0);
            for (int64_t p = s; p < e; ++p) seg[tile_of(P.kcol[p], tw, Tmax)]++;
            for (size_t j = 0; j < J; ++j) {
                int64_t used = 0;
                for (int32_t t = 0; t < Ts[j]; ++t)
                    if (seg[t]) { add(base[j] + t, seg[t]); used += seg[t]; }
                if (e - s - used) add(base[j] + Ts[j], e - s - used);
            }
        }
        #pragma omp critical
        for (size_t k = 0; k < loc.size(); ++k) small[k] += loc[k];
    }
    out.assign(J, {});
    for (size_t j = 0; j < J; ++j) {
        out[j].assign(Ts[j] + 1, {});
        for (int32_t t = 0; t <= Ts[j]; ++t) {
            const size_t slot = base[j] + t;
            for (int64_t l = cap - 1; l >= kSmall; --l)
                if (big[slot][l]) out[j][t].push_back({l, big[slot][l]});
            for (int64_t l = std::min<int64_t>(cap, kSmall) - 1; l >= 0; --l)
                if (small[slot * kSmall + l]) out[j][t].push_back({l, small[slot * kSmall + l]});
        }
    }
}

void tile_histograms(const Prepared& P, int64_t tw, int32_t T,
                     std::vector<std::vector<std::pair<int64_t, int64_t>>>& hist) {
    std::vector<std::vector<std::vector<std::pair<int64_t, int64_t>>>> out;
    tile_histograms_multi(P, tw, std::vector<int32_t>{T}, out);
    hist = std::move(out[0]);
}

spmv_status pack_layout(const Prepared& P, const BuildParams& bp, HostLayout& L) {
    const int64_t n = P.n_rows, tw = bp.tile_width;
    const int32_t T = bp.num_tiles;
    if (tw < 1 || T < 0 || (int64_t)bp.wl.size() != T + 1 || bp.align_rm < 1 || bp.ell_h < 1) {
        set_error("bad build parameters"); return SPMV_EINVAL;
    }
    if ((int64_t)T * tw > P.n_cols + tw - 1 && T > 0) { set_error("num_tiles exceeds ceil(n_cols / tile_width)"); return SPMV_ERANGE; }
    for (auto w : bp.wl) if (w < 1) { set_error("workload size must be >= 1"); return SPMV_EINVAL; }
    const int64_t align = bp.align_rm, eh = bp.ell_h;

    // first/last tile touched by every row (entries are ordered by relabelled column)
    std::vector<int32_t> first_t(n), last_t(n);
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        int64_t s = P.rp[i], e = P.rp[i + 1];
        first_t[i] = s < e ? tile_of(P.kcol[s], tw, T) : T;
        last_t[i] = s < e ? tile_of(P.kcol[e - 1], tw, T) : T;
    }
    std::vector<int64_t> cursor(P.rp.begin(), P.rp.end() - 1);
    std::vector<int64_t> seg_start(n);
    std::vector<int32_t> seg_len(n);
    L.tiles.assign(T + 1, TileInfo{});
    L.desc.clear(); L.row_id.clear(); L.slot_col.clear(); L.slot_val.clear(); L.split.clear();
    L.n_chunks = 0;
    int64_t n_slots = 0;

    for (int32_t t = 0; t <= T; ++t) {
        TileInfo& ti = L.tiles[t];
        ti.col_lo = std::min<int64_t>((int64_t)t * tw, P.n_cols);
        ti.col_hi = (t < T) ? std::min<int64_t>((int64_t)(t + 1) * tw, P.n_cols) : P.n_cols;
        const int64_t lo = ti.col_lo, hi = ti.col_hi;
        const int32_t sentinel = (int32_t)(hi - lo);
        const int64_t WL = bp.wl[t];
        ti.wl = (int32_t)WL;
        ti.wl_begin = (int64_t)L.desc.size();
        // a4: in-tile segment of every row
        int64_t maxlen = 0, tnnz = 0;
        #pragma omp parallel for schedule(static) reduction(max : maxlen) reduction(+ : tnnz)
        for (int64_t i = 0; i < n; ++i) {
            int64_t c = cursor[i], e = P.rp[i + 1];
            seg_start[i] = c;
            if (t < T) while (c < e && P.kcol[c] < hi) ++c;
            else c = e;
            seg_len[i] = (int32_t)(c - seg_start[i]);
            cursor[i] = c;
            maxlen = std::max<int64_t>(maxlen, c - seg_start[i]);
            tnnz += c - seg_start[i];
        }
        ti.nnz = tnnz;
        if (!bp.split && maxlen > WL) {
            set_error("workload size below the tile's longest row with split_long_rows = 0");
            return SPMV_EROWSPLIT;
        }
        // counting sort of touched rows by (length desc, id asc); zero rows last in the remainder
        std::vector<int64_t> bucket(maxlen + 2, 0);
        int64_t n_zero = 0;
        for (int64_t i = 0; i < n; ++i) {
            if (seg_len[i] > 0) bucket[maxlen - seg_len[i] + 1]++;
            else if (t == T && P.rp[i + 1] == P.rp[i]) ++n_zero;
        }
        for (int64_t b = 0; b <= maxlen; ++b) bucket[b + 1] += bucket[b];
        const int64_t n_nonzero_rows = bucket[maxlen + 1];
        std::vector<int32_t> rows(n_nonzero_rows + n_zero);
        {
            int64_t zpos = n_nonzero_rows;
            for (int64_t i = 0; i < n; ++i) {
                if (seg_len[i] > 0) rows[bucket[maxlen - seg_len[i]]++] = (int32_t)i;
                else if (t == T && P.rp[i + 1] == P.rp[i]) rows[zpos++] = (int32_t)i;
            }
        }
        ti.rows = (int64_t)rows.size();
        auto entry_of = [&](int32_t r) -> uint32_t {
            uint32_t e = (uint32_t)r;
            if (first_t[r] < t) e |= FLAG_ACC;
            if (last_t[r] <= t) e |= FLAG_FINAL;
            return e;
        };
        auto len_of = [&](int32_t r) -> int64_t { return seg_len[r]; };
        // a5: packing walk (Alg. 3 lines 7-15)
        const int64_t wl_first = (int64_t)L.desc.size();
        const int64_t nr = (int64_t)rows.size();
        int64_t i = 0;
        auto camp = [&](int64_t size) {
            if (bp.camping && size > 0 && size % 512 == 0) n_slots += 64;
        };
        // TILE-COO: the dense tiles as COO workloads, the remainder composite (R19)
        const bool coo = bp.orient == 3 && t < T;
        const int32_t orient_t = bp.orient == 3 ? 0 : bp.orient;
        while (i < nr) {
            int64_t w = len_of(rows[i]);
            int64_t hq = std::max<int64_t>(1, WL / std::max<int64_t>(w, 1));
            if (coo && !(bp.split && w > WL)) {
                // whole rows while the workload holds at most WL entries (at least one row), padded
                // to a multiple of 32 slots: a row never crosses a workload (one writer per row)
                int64_t h = 0, tot = 0;
                while (i + h < nr && (h == 0 || tot + len_of(rows[i + h]) <= WL)) tot += len_of(rows[i + h++]);
                const int64_t wp = roundup(tot, 32);
                L.desc.push_back(WlDesc{n_slots, (int32_t)L.row_id.size(), (int32_t)wp, (int32_t)h, KIND_COO, 1, 0, -1, 0});
                for (int64_t r = 0; r < h; ++r) L.row_id.push_back(entry_of(rows[i + r]));
                n_slots += wp;
                camp(wp);
                i += h;
                continue;
            }
            if (bp.split && w > WL) {
                int32_t r = rows[i];
                int64_t nch = (w + WL - 1) / WL;
                int32_t sid = (int32_t)(L.split.size() / 3);
                L.split.push_back((int32_t)entry_of(r));
                L.split.push_back((int32_t)nch);
                L.split.push_back((int32_t)L.n_chunks);
                L.n_chunks += nch;
                for (int64_t c = 0; c < nch; ++c) {
                    int64_t part = std::min<int64_t>(WL, w - c * WL);
                    int64_t wp = roundup(part, align);
                    L.desc.push_back(WlDesc{n_slots, (int32_t)L.row_id.size(), (int32_t)wp, 1, KIND_SPLIT, 4, 0, sid, (int32_t)c});
                    L.row_id.push_back(entry_of(r));
                    n_slots += wp;
                    camp(wp);
                }
                ++i;
                continue;
            }
            if (row_major(orient_t, w, hq)) {
                int64_t h = std::min<int64_t>(hq, nr - i);
                int64_t wp = roundup(w, align);
                L.desc.push_back(WlDesc{n_slots, (int32_t)L.row_id.size(), (int32_t)wp, (int32_t)h, KIND_RM, 4, 0, -1, 0});
                for (int64_t r = 0; r < h; ++r) L.row_id.push_back(entry_of(rows[i + r]));
                n_slots += h * wp;
                camp(h * wp);
                i += h;
            } else {
                int64_t hp = roundup(hq, eh);
                int64_t take = std::min<int64_t>(hp, nr - i);
                int64_t slabs = (take + eh - 1) / eh;
                uint8_t kvec = (w % 4 == 0) ? 4 : ((w % 2 == 0) ? 2 : 1);
                if (ti.threshold == 0 && w > 0) ti.threshold = (int32_t)w;
                L.desc.push_back(WlDesc{n_slots, (int32_t)L.row_id.size(), (int32_t)w, (int32_t)(slabs * eh), KIND_CM, kvec, 0, -1, 0});
                for (int64_t r = 0; r < slabs * eh; ++r)
                    L.row_id.push_back(r < take ? entry_of(rows[i + r]) : PAD_ROW);
                n_slots += slabs * eh * w;
                camp(slabs * eh * w);
                i += take;
            }
        }
        ti.wl_end = (int64_t)L.desc.size();
        // descriptors address row entries and split partials with int32 (WlDesc::row_base, split table)
        if ((int64_t)L.row_id.size() > (int64_t)INT32_MAX || L.n_chunks > (int64_t)INT32_MAX) {
            set_error("more than 2^31-1 row entries or split chunks: use fewer tiles or a larger workload size");
            return SPMV_ERANGE;
        }
        // fill slots (parallel over this tile's workloads); rows of RM/CM workloads are
        // consecutive in `rows`, recovered from row_id entries
        L.slot_col.resize(n_slots, sentinel);
        if (!P.pattern) L.slot_val.resize(n_slots, 0.0f);
        // dead space (camping pad / padding) must hold the sentinel of *this* tile
        const int64_t tile_slot_lo = L.desc.size() > (size_t)wl_first ? L.desc[wl_first].off : n_slots;
        #pragma omp parallel for schedule(static)
        for (int64_t s = tile_slot_lo; s < n_slots; ++s) {
            L.slot_col[s] = sentinel;
            if (!P.pattern) L.slot_val[s] = 0.0f;
        }
        ti.slots = n_slots - tile_slot_lo;
        #pragma omp parallel for schedule(dynamic, 64)
        for (int64_t j = wl_first; j < (int64_t)L.desc.size(); ++j) {
            const WlDesc& d = L.desc[j];
            if (d.kind == KIND_SPLIT) {
                int32_t r = (int32_t)(L.row_id[d.row_base] & ROW_MASK);
                int64_t src = seg_start[r] + (int64_t)d.chunk * WL;
                int64_t part = std::min<int64_t>(WL, seg_len[r] - (int64_t)d.chunk * WL);
                for (int64_t k = 0; k < part; ++k) {
                    L.slot_col[d.off + k] = (int32_t)(P.kcol[src + k] - lo);
                    if (!P.pattern) L.slot_val[d.off + k] = P.kval[src + k];
                }
            } else if (d.kind == KIND_COO) {
                int64_t dst = d.off;
                for (int32_t rr = 0; rr < d.h; ++rr) {
                    int32_t r = (int32_t)(L.row_id[d.row_base + rr] & ROW_MASK);
                    int64_t src = seg_start[r], cnt = seg_len[r];
                    for (int64_t k = 0; k < cnt; ++k) {
                        L.slot_col[dst + k] = (int32_t)((uint32_t)(P.kcol[src + k] - lo) | (k + 1 == cnt ? COO_END : 0u));
                        if (!P.pattern) L.slot_val[dst + k] = P.kval[src + k];
                    }
                    dst += cnt;
                }
            } else if (d.kind == KIND_RM) {
                for (int32_t rr = 0; rr < d.h; ++rr) {
                    int32_t r = (int32_t)(L.row_id[d.row_base + rr] & ROW_MASK);
                    int64_t src = seg_start[r], cnt = seg_len[r];
                    int64_t dst = d.off + (int64_t)rr * d.w;
                    for (int64_t k = 0; k < cnt; ++k) {
                        L.slot_col[dst + k] = (int32_t)(P.kcol[src + k] - lo);
                        if (!P.pattern) L.slot_val[dst + k] = P.kval[src + k];
                    }
                }
            } else {
                const int64_t kv = d.kvec;
                for (int32_t rr = 0; rr < d.h; ++rr) {
                    uint32_t e = L.row_id[d.row_base + rr];
                    if (e == PAD_ROW) continue;
                    int32_t r = (int32_t)(e & ROW_MASK);
                    int64_t src = seg_start[r], cnt = seg_len[r];
                    int64_t slab_off = d.off + (int64_t)(rr / eh) * eh * d.w;
                    int64_t lr = rr % eh;
                    for (int64_t k = 0; k < cnt; ++k) {
                        int64_t pos = slab_off + (k / kv) * eh * kv + lr * kv + (k % kv);
                        L.slot_col[pos] = (int32_t)(P.kcol[src + k] - lo);
                        if (!P.pattern) L.slot_val[pos] = P.kval[src + k];
                    }
                }
            }
        }
    }
    return SPMV_OK;
}

}  // namespace tc
