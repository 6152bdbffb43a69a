// graph_build.h -- host construction of the iteration matrices (App. F): adjacency
// clean-up, transposes, symmetric relabelling by column length.
#pragma once
#include <algorithm>
#ifdef _OPENMP
#include <omp.h>
#endif
#include <cstdint>
#include <vector>

namespace tc {

// ------------------------------------------------------------------ host: graph matrices
// counting sort permutation of [0,N) by (len desc, id asc): pi[id] = new position
inline void order_by_length(const std::vector<int64_t>& len, std::vector<int32_t>& pi) {
    const int64_t N = (int64_t)len.size();
    int64_t mx = 0;
    for (auto l : len) mx = std::max(mx, l);
    std::vector<int64_t> start(mx + 2, 0);
    for (auto l : len) start[mx - l + 1]++;
    for (int64_t b = 0; b <= mx; ++b) start[b + 1] += start[b];
    pi.assign(N, 0);
    for (int64_t i = 0; i < N; ++i) pi[i] = (int32_t)start[mx - len[i]]++;
}

// dedupe each row of an adjacency CSR (sorted unique targets per row)
inline void clean_adjacency(int64_t n, const int64_t* rp, const int32_t* col,
                            std::vector<int64_t>& orp, std::vector<int32_t>& ocol) {
    std::vector<int64_t> len(n);
    ocol.assign(col, col + rp[n]);
    #pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t u = 0; u < n; ++u) {
        int32_t* b = ocol.data() + rp[u];
        int32_t* e = ocol.data() + rp[u + 1];
        std::sort(b, e);
        len[u] = std::unique(b, e) - b;
    }
    orp.assign(n + 1, 0);
    for (int64_t u = 0; u < n; ++u) orp[u + 1] = orp[u] + len[u];
    std::vector<int32_t> packed(orp[n]);
    #pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t u = 0; u < n; ++u)
        std::copy(ocol.begin() + rp[u], ocol.begin() + rp[u] + len[u], packed.begin() + orp[u]);
    ocol.swap(packed);
}

// relabelled CSR of a matrix given as a list of (row, col) by a generator callback over rows
struct Coo { std::vector<int64_t> rp; std::vector<int32_t> col; };

// rows of the relabelled matrix: entries of original row r go to row pi[r], cols mapped by pi
inline void relabel_csr(int64_t N, const std::vector<int64_t>& rp, const std::vector<int32_t>& col,
                        const std::vector<int32_t>& pi, Coo& out) {
    out.rp.assign(N + 1, 0);
    for (int64_t r = 0; r < N; ++r) out.rp[pi[r] + 1] = rp[r + 1] - rp[r];
    for (int64_t i = 0; i < N; ++i) out.rp[i + 1] += out.rp[i];
    out.col.resize(rp[N]);
    #pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t r = 0; r < N; ++r) {
        int64_t d = out.rp[pi[r]];
        for (int64_t k = rp[r]; k < rp[r + 1]; ++k) out.col[d++] = pi[col[k]];
    }
}

// transpose of an n x n pattern CSR (row v lists sources u ascending)
// Parallel without atomics: thread j owns the target rows [v_j, v_{j+1}) and scans every entry in
// source order, so each output row lists its sources ascending (the serial order) -- T read passes
// over col instead of contended atomic counters on the hub rows.
inline void transpose(int64_t n, const std::vector<int64_t>& rp, const std::vector<int32_t>& col,
                      std::vector<int64_t>& trp, std::vector<int32_t>& tcol) {
    trp.assign(n + 1, 0);
    const int64_t m = rp[n];
    int T = 1;
#ifdef _OPENMP
    T = std::max(1, omp_get_max_threads());
#endif
    if (m < (int64_t)1 << 20) T = 1;
    std::vector<int64_t> vb(T + 1);
    for (int j = 0; j <= T; ++j) vb[j] = n * j / T;
    #pragma omp parallel for num_threads(T) schedule(static, 1)
    for (int j = 0; j < T; ++j)
        for (int64_t k = 0; k < m; ++k) {
            const int32_t v = col[k];
            if (v >= vb[j] && v < vb[j + 1]) trp[v + 1]++;
        }
    for (int64_t i = 0; i < n; ++i) trp[i + 1] += trp[i];
    // scatter ranges balanced by entry count
    for (int j = 1; j < T; ++j)
        vb[j] = std::upper_bound(trp.begin(), trp.end(), m * j / T) - trp.begin() - 1;
    for (int j = 1; j <= T; ++j) vb[j] = std::max(vb[j], vb[j - 1]);
    vb[T] = n;
    tcol.resize(m);
    std::vector<int64_t> pos(trp.begin(), trp.end() - 1);
    #pragma omp parallel for num_threads(T) schedule(static, 1)
    for (int j = 0; j < T; ++j)
        for (int64_t u = 0; u < n; ++u)
            for (int64_t k = rp[u]; k < rp[u + 1]; ++k) {
                const int32_t v = col[k];
                if (v >= vb[j] && v < vb[j + 1]) tcol[pos[v]++] = (int32_t)u;
            }
}

// Iteration matrix M of each algorithm in original vertex ids, and its column lengths:
//   algo 0 PageRank: M = A^T (row v lists sources u of u -> v), column u length = outdeg(u)
//   algo 2 RWR:      M = binary(A u A^T), symmetric, column length = degree
//   algo 1 HITS:     M = [[0, A^T], [A, 0]] on 2n indices (Eq. 8)
// Returns the vector length N (n or 2n).
inline int64_t build_iteration_matrix(int algo, int64_t n, const std::vector<int64_t>& arp,
                                      const std::vector<int32_t>& acol, std::vector<int64_t>& mrp,
                                      std::vector<int32_t>& mcol, std::vector<int64_t>& len) {
    if (algo == 0) {
        transpose(n, arp, acol, mrp, mcol);
        len.resize(n);
        for (int64_t u = 0; u < n; ++u) len[u] = arp[u + 1] - arp[u];
        return n;
    }
    std::vector<int64_t> trp; std::vector<int32_t> tcol;
    transpose(n, arp, acol, trp, tcol);
    if (algo == 2) {
        mrp.assign(n + 1, 0);
        std::vector<int64_t> slen(n);
        #pragma omp parallel
        {
            std::vector<int32_t> buf;
            #pragma omp for schedule(dynamic, 1024)
            for (int64_t i = 0; i < n; ++i) {
                buf.assign(acol.begin() + arp[i], acol.begin() + arp[i + 1]);
                buf.insert(buf.end(), tcol.begin() + trp[i], tcol.begin() + trp[i + 1]);
                std::sort(buf.begin(), buf.end());
                slen[i] = std::unique(buf.begin(), buf.end()) - buf.begin();
            }
        }
        for (int64_t i = 0; i < n; ++i) mrp[i + 1] = mrp[i] + slen[i];
        mcol.resize(mrp[n]);
        #pragma omp parallel
        {
            std::vector<int32_t> buf;
            #pragma omp for schedule(dynamic, 1024)
            for (int64_t i = 0; i < n; ++i) {
                buf.assign(acol.begin() + arp[i], acol.begin() + arp[i + 1]);
                buf.insert(buf.end(), tcol.begin() + trp[i], tcol.begin() + trp[i + 1]);
                std::sort(buf.begin(), buf.end());
                buf.erase(std::unique(buf.begin(), buf.end()), buf.end());
                std::copy(buf.begin(), buf.end(), mcol.begin() + mrp[i]);
            }
        }
        len.resize(n);
        for (int64_t u = 0; u < n; ++u) len[u] = mrp[u + 1] - mrp[u];
        return n;
    }
    const int64_t N = 2 * n;
    mrp.assign(N + 1, 0);
    for (int64_t v = 0; v < n; ++v) mrp[v + 1] = trp[v + 1] - trp[v];
    for (int64_t u = 0; u < n; ++u) mrp[n + u + 1] = arp[u + 1] - arp[u];
    for (int64_t i = 0; i < N; ++i) mrp[i + 1] += mrp[i];
    mcol.resize(mrp[N]);
    #pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t v = 0; v < n; ++v) {
        int64_t d = mrp[v];
        for (int64_t k = trp[v]; k < trp[v + 1]; ++k) mcol[d++] = (int32_t)(n + tcol[k]);
    }
    #pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t u = 0; u < n; ++u) {
        int64_t d = mrp[n + u];
        for (int64_t k = arp[u]; k < arp[u + 1]; ++k) mcol[d++] = acol[k];
    }
    len.assign(N, 0);
    for (int64_t k = 0; k < mrp[N]; ++k) len[mcol[k]]++;
    return N;
}

}  // namespace tc
