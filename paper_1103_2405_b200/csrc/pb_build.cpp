// pb_build.cpp -- host builder of the two-phase tile layout (pb.h).
//
//   bins    consecutive rows, region (products) <= rcap, position block <= pcap, <= kMaxRows rows;
//           a row longer than rcap is a bin of its own (PB_LONG: summed by streaming, no positions).
//           Inside a bin rows are ranked by (length desc, id asc) (Observation 5) and
//           split at the composite threshold `heavy` (Solution 3, L88): longer rows are warp-per-row
//           with contiguous positions (CSR-vector, L80-L82), shorter rows thread-per-row over
//           32-row slabs whose positions are column major (ELL, L84; slab width = its first row).
//   groups  consecutive bins, regions <= gcap products.
//   chunks  per group: the group's entries in column order (counting sort, "linear time", L98),
//           cut every ccap entries / xcap columns / nrcap distinct bins (Solution 1's tile of x,
//           L56-L60, sized for shared memory); inside a chunk entries are re-ordered by (bin,
//           column, row) so that each bin's entries ("run") are contiguous and land contiguously in
//           the bin's region.
#include <algorithm>
#include <cstring>
#include <numeric>
#include <string>

#include "pb.h"
#include "plan.h"

namespace tc {

static inline int64_t rup(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

// staged bytes of an item, each stream from the 16-byte boundary at or below its first element
int64_t pb_chunk_bytes(const PbChunk& c, bool valued) {
    const int64_t e = 4 * rup((c.e0 & 3) + c.n, 4);
    return e * (valued ? 2 : 1) + 4 * rup((c.col0 & 3) + c.span, 4) + 4 * rup((c.run0 & 3) + c.nrun, 4);
}
int64_t pb_bin_bytes(const PbBin& b) {
    if (b.kind == PB_LONG) return 2 * 4 * rup((b.row0 & 3) + 1, 4);
    return 4 * rup(b.rlen, 4) + 2 * (int64_t)b.plen + 2 * 4 * rup((b.row0 & 3) + b.nrows, 4);
}

int64_t pb_stage_bytes(const PbLayout& L) {
    int64_t mx = 16;
    for (const auto& c : L.chunks) mx = std::max(mx, pb_chunk_bytes(c, !L.pattern));
    for (const auto& b : L.bins) mx = std::max(mx, pb_bin_bytes(b));
    return 128 + rup(mx, 128);
}

// rows of bin [r0, r1) ranked by (length desc, id asc)
static void rank_rows(const std::vector<int64_t>& len, int64_t r0, int64_t r1, std::vector<int64_t>& order) {
    order.resize(r1 - r0);
    std::iota(order.begin(), order.end(), r0);
    std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return len[a] > len[b]; });
}

// position block length of a ranked bin: heavy rows contiguous, light rows in 32-row slabs of the
// slab's first (longest) length
static int64_t pos_len(const std::vector<int64_t>& len, const std::vector<int64_t>& order, int32_t heavy) {
    int64_t p = 0, i = 0;
    const int64_t n = (int64_t)order.size();
    for (; i < n && len[order[i]] >= heavy; ++i) p += len[order[i]];
    for (; i < n; i += 32) p += 32 * len[order[i]];
    return rup(p, 8);
}

bool pb_build(int64_t n_rows, int64_t n_cols, const int64_t* rp, const int32_t* col, const float* val,
              bool pattern, const PbParams& prm, PbLayout& L) {
    if (prm.rcap < 32 || prm.rcap > 65535 || prm.maxrows < 1 || prm.pcap < 1024 || prm.pcap > 65535 || prm.xcap < 1 ||
        prm.xcap > 65536 || prm.ccap < 1 || prm.nrcap < 1 || prm.nrcap > 65536 || prm.heavy < 1 ||
        prm.gcap < 1) {
        set_error("two-phase parameters out of range"); return false;
    }
    L = PbLayout();
    L.n_rows = n_rows; L.n_cols = n_cols; L.nnz = n_rows ? rp[n_rows] : 0; L.pattern = pattern; L.prm = prm;
    std::vector<int64_t> len(n_rows);
    for (int64_t i = 0; i < n_rows; ++i) len[i] = rp[i + 1] - rp[i];

    // ---- bins
    struct B { int64_t r0, r1; bool lng; };
    std::vector<B> bins;
    std::vector<int64_t> order;
    for (int64_t r = 0; r < n_rows;) {
        if (len[r] > prm.rcap) { bins.push_back({r, r + 1, true}); ++r; continue; }
        int64_t r1 = r, reg = 0;
        while (r1 < n_rows && len[r1] <= prm.rcap && reg + len[r1] <= prm.rcap && r1 - r < prm.maxrows) reg += len[r1++];
        for (;;) {
            rank_rows(len, r, r1, order);
            if (pos_len(len, order, prm.heavy) <= prm.pcap || r1 == r + 1) break;
            r1 = r + std::max<int64_t>(1, (r1 - r) / 2);
        }
        bins.push_back({r, r1, false});
        r = r1;
    }
    const int64_t nb = (int64_t)bins.size();
    if (nb >= (int64_t(1) << 31) - 1) { set_error("too many bins"); return false; }

    // ---- groups, regions, row order, position blocks
    L.bins.resize(nb);
    std::vector<int64_t> bin_group(nb);
    std::vector<int64_t> g_bin0;            // first bin of each group
    int64_t roff = 0, poff = 0, gsum = 0, pr = 0;
    std::vector<int32_t> binof(n_rows);
    std::vector<int64_t> pbase(n_rows, -1); // global pos index of a row's first product
    std::vector<int8_t> pstride(n_rows, 0);
    L.prow.resize(n_rows);
    L.pmeta.resize(n_rows);
    for (int64_t b = 0; b < nb; ++b) {
        const B& bb = bins[b];
        int64_t rl = 0;
        for (int64_t r = bb.r0; r < bb.r1; ++r) rl += len[r];
        const int64_t alloc = rup(rl, 32);     // whole 128-byte lines: a consumed region is discarded from L2
        if (g_bin0.empty() || (gsum > 0 && gsum + alloc > prm.gcap)) { g_bin0.push_back(b); gsum = 0; }
        gsum += alloc;
        PbBin& d = L.bins[b];
        d.roff = roff; d.rlen = (int32_t)std::min<int64_t>(rl, INT32_MAX);
        if (rl > INT32_MAX) { set_error("row longer than 2^31 entries"); return false; }
        d.row0 = pr; d.nrows = (int32_t)(bb.r1 - bb.r0);
        d.group = (int32_t)(g_bin0.size() - 1);
        d.kind = bb.lng ? PB_LONG : PB_BIN;
        d.poff = poff;
        bin_group[b] = d.group;
        roff += alloc;
        if (bb.lng) {
            d.plen = 0; d.nheavy = 1;
            L.prow[pr] = (uint32_t)bb.r0 | FLAG_FINAL;
            L.pmeta[pr] = 0;
            binof[bb.r0] = (int32_t)b;
            ++pr;
            continue;
        }
        rank_rows(len, bb.r0, bb.r1, order);
        const int64_t n = (int64_t)order.size();
        int64_t i = 0, p = 0;
        for (; i < n && len[order[i]] >= prm.heavy; ++i) {
            const int64_t r = order[i];
            L.prow[pr + i] = (uint32_t)r | FLAG_FINAL;
            L.pmeta[pr + i] = (uint32_t)p | ((uint32_t)len[r] << 16);
            pbase[r] = poff + p; pstride[r] = 1;
            p += len[r];
        }
        d.nheavy = (int32_t)i;
        for (int64_t s0 = i; s0 < n; s0 += 32) {
            const int64_t w = len[order[s0]];
            for (int64_t l = 0; l < 32 && s0 + l < n; ++l) {
                const int64_t r = order[s0 + l];
                L.prow[pr + s0 + l] = (uint32_t)r | FLAG_FINAL;
                L.pmeta[pr + s0 + l] = (uint32_t)(p + l) | ((uint32_t)len[r] << 16);
                pbase[r] = poff + p + l; pstride[r] = 32;
            }
            p += 32 * w;
        }
        d.plen = (int32_t)rup(p, 8);
        for (int64_t r = bb.r0; r < bb.r1; ++r) binof[r] = (int32_t)b;
        poff += d.plen;
        pr += n;
    }
    L.buf_floats = std::max<int64_t>(roff, 4);
    L.pos.assign(std::max<int64_t>(poff, 8), 0);
    const int64_t G = (int64_t)g_bin0.size();
    L.n_groups = (int32_t)G;
    g_bin0.push_back(nb);

    // ---- chunks per group (groups are independent: row ranges and entry ranges are disjoint)
    L.cd.resize(L.nnz);
    if (!pattern) L.val.resize(L.nnz);
    std::vector<std::vector<PbChunk>> gch(G);
    std::vector<std::vector<int32_t>> grun(G);
    bool ok = true;
    #pragma omp parallel
    {
        std::vector<int64_t> cstart;
        std::vector<int32_t> crow;
        std::vector<float> cval;
        std::vector<int64_t> last_chunk, fill, run_at;
        std::vector<int32_t> cbins, ccol, cr;
        std::vector<float> cv;
        #pragma omp for schedule(dynamic, 1)
        for (int64_t g = 0; g < G; ++g) {
            const int64_t b0 = g_bin0[g], b1 = g_bin0[g + 1];
            const int64_t R0 = bins[b0].r0, R1 = bins[b1 - 1].r1;
            const int64_t E0 = rp[R0], E1 = rp[R1], mg = E1 - E0;
            const int64_t gbase = L.bins[b0].roff;
            // counting sort of the group's entries by column (rows ascending within a column)
            cstart.assign(n_cols + 1, 0);
            for (int64_t k = E0; k < E1; ++k) cstart[col[k] + 1]++;
            for (int64_t j = 0; j < n_cols; ++j) cstart[j + 1] += cstart[j];
            crow.resize(mg);
            if (!pattern) cval.resize(mg);
            {
                std::vector<int64_t> f(cstart.begin(), cstart.end() - 1);
                for (int64_t r = R0; r < R1; ++r)
                    for (int64_t k = rp[r]; k < rp[r + 1]; ++k) {
                        const int64_t q = f[col[k]]++;
                        crow[q] = (int32_t)r;
                        if (!pattern) cval[q] = val[k];
                    }
            }
            last_chunk.assign(b1 - b0, -1);
            fill.assign(b1 - b0, 0);
            run_at.assign(b1 - b0, -1);
            std::vector<PbChunk>& chunks = gch[g];
            std::vector<int32_t>& runs = grun[g];
            int64_t e_out = E0;                     // next output entry (global index)
            // sweep columns; a chunk is [q0, q1) of the column-ordered entries
            int64_t q = 0, j = 0;
            while (q < mg) {
                while (cstart[j + 1] <= q) ++j;    // column of entry q
                const int64_t q0 = q, col0 = j;
                const int64_t cid = (int64_t)chunks.size();
                cbins.clear();
                int64_t jj = j;
                while (q < mg) {
                    while (cstart[jj + 1] <= q) ++jj;
                    if (q - q0 == prm.ccap || jj - col0 + 1 > prm.xcap) break;
                    const int64_t bl = binof[crow[q]] - b0;
                    if (last_chunk[bl] != cid) {
                        if ((int64_t)cbins.size() == prm.nrcap) break;
                        last_chunk[bl] = cid;
                        cbins.push_back((int32_t)bl);
                    }
                    ++q;
                }
                const int64_t q1 = q;
                int64_t last_col = col0;
                {
                    int64_t t = j;
                    while (cstart[t + 1] < q1) ++t;
                    last_col = t;
                }
                std::sort(cbins.begin(), cbins.end());
                // runs in bin order; counting placement (stable: column, row order kept)
                const int64_t nrun = (int64_t)cbins.size();
                std::vector<int64_t> rcount(nrun + 1, 0);
                for (int64_t i = 0; i < nrun; ++i) run_at[cbins[i]] = i;
                for (int64_t t = q0; t < q1; ++t) rcount[run_at[binof[crow[t]] - b0] + 1]++;
                for (int64_t i = 0; i < nrun; ++i) rcount[i + 1] += rcount[i];
                PbChunk ch{};
                ch.e0 = e_out; ch.gbase = gbase; ch.run0 = (int64_t)runs.size();
                ch.n = (int32_t)(q1 - q0); ch.col0 = (int32_t)col0; ch.span = (int32_t)(last_col - col0 + 1);
                ch.nrun = (int32_t)nrun; ch.group = (int32_t)g;
                std::vector<int64_t> rfill0(nrun);
                for (int64_t i = 0; i < nrun; ++i) {
                    const int64_t bl = cbins[i];
                    const PbBin& bd = L.bins[b0 + bl];
                    rfill0[i] = fill[bl];
                    const int64_t dest_first = bd.roff - gbase + fill[bl];
                    const int64_t d = dest_first - rcount[i];
                    if (d > INT32_MAX || d < INT32_MIN) { ok = false; }
                    runs.push_back((int32_t)d);
                    fill[bl] += rcount[i + 1] - rcount[i];
                }
                std::vector<int64_t> rpos(rcount.begin(), rcount.end() - 1);
                int64_t t_col = j;
                for (int64_t t = q0; t < q1; ++t) {
                    while (cstart[t_col + 1] <= t) ++t_col;
                    const int32_t r = crow[t];
                    const int64_t bl = binof[r] - b0;
                    const int64_t ri = run_at[bl];
                    const int64_t loc = rpos[ri]++;
                    const int64_t e = e_out + loc;
                    L.cd[e] = (uint32_t)(t_col - col0) | ((uint32_t)ri << 16);
                    if (!pattern) L.val[e] = cval[t];
                    // region position of this product and its slot in the row's position list
                    const int64_t qreg = rfill0[ri] + (loc - rcount[ri]);
                    if (pstride[r]) {
                        // rows are visited column by column: the row's t-th product is its t-th visit
                        int64_t& pb = pbase[r];
                        L.pos[pb] = (uint16_t)qreg;
                        pb += pstride[r];
                    }
                }
                e_out += q1 - q0;
                chunks.push_back(ch);
            }
        }
    }
    if (!ok) { set_error("two-phase run offset exceeds 2^31"); return false; }
    // ---- concatenate per-group chunk lists; work queue E0 E1 R0 E2 R1 ... R(G-1)
    int64_t run_base = 0;
    std::vector<int64_t> gc0(G + 1, 0);
    for (int64_t g = 0; g < G; ++g) {
        for (auto& c : gch[g]) { c.run0 += run_base; L.chunks.push_back(c); }
        L.runs.insert(L.runs.end(), grun[g].begin(), grun[g].end());
        run_base += (int64_t)grun[g].size();
        gc0[g + 1] = (int64_t)L.chunks.size();
        L.group_chunks.push_back((int32_t)gch[g].size());
    }
    if ((int64_t)L.chunks.size() >= (int64_t(1) << 31) - 1) { set_error("too many chunks"); return false; }
    auto push_e = [&](int64_t g) { for (int64_t c = gc0[g]; c < gc0[g + 1]; ++c) L.items.push_back((int32_t)c); };
    auto push_r = [&](int64_t g) { for (int64_t b = g_bin0[g]; b < g_bin0[g + 1]; ++b) L.items.push_back(~(int32_t)b); };
    for (int64_t g = 0; g < G; ++g) {
        push_e(g);
        if (g >= 1) push_r(g - 1);
    }
    if (G > 0) push_r(G - 1);
    if (L.runs.empty()) L.runs.push_back(0);
    L.stage_bytes = pb_stage_bytes(L);
    return true;
}

bool pb_build_fit(int64_t n_rows, int64_t n_cols, const int64_t* rp, const int32_t* col, const float* val,
                  bool pattern, PbParams prm, bool xcap_fixed, PbLayout& L) {
    if (!pb_build(n_rows, n_cols, rp, col, val, pattern, prm, L)) return false;
    if (xcap_fixed || prm.xcap <= kPbXcapFallback || 2 * L.stage_bytes <= kPbTwoCtaSmem) return true;
    prm.xcap = kPbXcapFallback;
    L = PbLayout();
    return pb_build(n_rows, n_cols, rp, col, val, pattern, prm, L);
}

}  // namespace tc
