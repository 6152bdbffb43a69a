/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY.  Plain, slow, obviously-correct fp64 CPU reference for
 * the tiled-composite SpMV path of Yang, Parthasarathy & Sadayappan (VLDB 2011).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
 * load this library.  It shares no code, header, table or helper with the product library
 * (paper_1103_2405_b200/); it is compiled separately and neither side includes the other.
 *
 * Every routine is the plain definition written out, in fp64, summing left to right:
 *   oracle_spmv      y = A x                                  PAPER.md L291 (App. B problem statement)
 *   oracle_pagerank  p(k+1) = c W^T p(k) + (1-c) p(0)         PAPER.md L414-L416, L430 (Eq. 6)
 *                    with dangling mass redistributed uniformly (reading R1)
 *   oracle_hits      [a;h](k+1) = [[0,A^T],[A,0]] [a;h](k)    PAPER.md L432-L440 (Eq. 7-8)
 *                    halves normalised separately (L2 default, L1 = "sum to 1", reading R3)
 *   oracle_rwr       r(k+1) = c W r(k) + (1-c) e_q            PAPER.md L452-L456 (Eq. 9)
 *                    W = column-normalised binary(A u A^T)     (readings R6-R8)
 * Convergence: L1 norm of the change < tol (reading R2); fixed_iters > 0 runs exactly that many
 * iterations instead (parity at the same k, reading R14).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

#define OR_EXPORT __attribute__((visibility("default")))

/* y_i = sum_k val[k] * x[col[k]] over row i's entries, left to right, in fp64.
 * b_i = sum_k |val[k] * x[col[k]]|  (the per-element tolerance scale).  val == NULL: pattern (1.0). */
OR_EXPORT void oracle_spmv(int64_t n_rows, const int64_t* row_ptr, const int32_t* col,
                           const float* val, const float* x, double* y, double* b) {
    #pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t i = 0; i < n_rows; ++i) {
        double s = 0.0, a = 0.0;
        for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
            double v = val ? (double)val[k] : 1.0;
            double t = v * (double)x[col[k]];
            s += t;
            a += fabs(t);
        }
        y[i] = s;
        if (b) b[i] = a;
    }
}

/* same, x given in fp64 (used by the power iterations below) */
static void spmv_d(int64_t n_rows, const int64_t* row_ptr, const int32_t* col,
                   const double* x, double* y) {
    #pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t i = 0; i < n_rows; ++i) {
        double s = 0.0;
        for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) s += x[col[k]];
        y[i] = s;
    }
}

/* transpose of a pattern CSR (n x n): row v of the result lists the sources u of edges u->v */
static void transpose_pattern(int64_t n, const int64_t* rp, const int32_t* col,
                              int64_t* trp, int32_t* tcol) {
    memset(trp, 0, (size_t)(n + 1) * sizeof(int64_t));
    for (int64_t k = 0; k < rp[n]; ++k) trp[col[k] + 1]++;
    for (int64_t i = 0; i < n; ++i) trp[i + 1] += trp[i];
    int64_t* pos = (int64_t*)malloc((size_t)n * sizeof(int64_t));
    memcpy(pos, trp, (size_t)n * sizeof(int64_t));
    for (int64_t u = 0; u < n; ++u)
        for (int64_t k = rp[u]; k < rp[u + 1]; ++k) tcol[pos[col[k]]++] = (int32_t)u;
    free(pos);
}

static double l1diff(int64_t n, const double* a, const double* b) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += fabs(a[i] - b[i]);
    return s;
}

/* PageRank, Eq. 6.  Input: adjacency A of G as CSR (row u lists the targets v of u->v).
 * W = row-normalised A; (W^T p)_v = sum over edges u->v of p_u / outdeg(u).
 * Dangling vertices (outdeg 0) spread their mass uniformly: + D/n with D = sum_{dangling} p_j.
 * p(0) = 1/n.  Returns 0, or 1 when max_iter was reached without convergence. */
OR_EXPORT int oracle_pagerank(int64_t n, const int64_t* row_ptr, const int32_t* col, double c,
                              double tol, int32_t max_iter, int32_t fixed_iters,
                              double* p_out, int32_t* iters_out, double* residual_out) {
    int64_t m = row_ptr[n];
    int64_t* trp = (int64_t*)malloc((size_t)(n + 1) * sizeof(int64_t));
    int32_t* tcol = (int32_t*)malloc((size_t)(m > 0 ? m : 1) * sizeof(int32_t));
    transpose_pattern(n, row_ptr, col, trp, tcol);
    double* p = (double*)malloc((size_t)n * sizeof(double));
    double* z = (double*)malloc((size_t)n * sizeof(double));
    double* y = (double*)malloc((size_t)n * sizeof(double));
    double* pn = (double*)malloc((size_t)n * sizeof(double));
    for (int64_t i = 0; i < n; ++i) p[i] = 1.0 / (double)n;
    int32_t it = 0; double res = INFINITY; int rc = 1;
    int32_t limit = fixed_iters > 0 ? fixed_iters : max_iter;
    while (it < limit) {
        double D = 0.0;
        for (int64_t u = 0; u < n; ++u) {
            int64_t od = row_ptr[u + 1] - row_ptr[u];
            if (od == 0) { D += p[u]; z[u] = 0.0; }
            else z[u] = p[u] / (double)od;
        }
        spmv_d(n, trp, tcol, z, y);                       /* y = W^T p */
        for (int64_t v = 0; v < n; ++v)
            pn[v] = c * (y[v] + D / (double)n) + (1.0 - c) / (double)n;
        res = l1diff(n, pn, p);
        memcpy(p, pn, (size_t)n * sizeof(double));
        ++it;
        if (fixed_iters <= 0 && res < tol) { rc = 0; break; }
    }
    if (fixed_iters > 0) rc = 0;
    memcpy(p_out, p, (size_t)n * sizeof(double));
    *iters_out = it; *residual_out = res;
    free(trp); free(tcol); free(p); free(z); free(y); free(pn);
    return rc;
}

/* normalise v in place: norm = 2 -> unit L2, norm = 1 -> sum of |v| = 1.  A zero vector becomes
 * uniform (reading R5); returns 1 in that case. */
static int normalise(int64_t n, double* v, int norm) {
    double s = 0.0;
    if (norm == 2) { for (int64_t i = 0; i < n; ++i) s += v[i] * v[i]; s = sqrt(s); }
    else { for (int64_t i = 0; i < n; ++i) s += fabs(v[i]); }
    if (s == 0.0) {
        double u = (norm == 2) ? 1.0 / sqrt((double)n) : 1.0 / (double)n;
        for (int64_t i = 0; i < n; ++i) v[i] = u;
        return 1;
    }
    for (int64_t i = 0; i < n; ++i) v[i] /= s;
    return 0;
}

/* HITS, Eq. 8 (simultaneous/Jacobi update): a' = A^T h, h' = A a; each half normalised;
 * a(0) = h(0) = 1/|V|; residual = |a'-a|_1 + |h'-h|_1 after normalisation. */
OR_EXPORT int oracle_hits(int64_t n, const int64_t* row_ptr, const int32_t* col, int32_t norm,
                          double tol, int32_t max_iter, int32_t fixed_iters,
                          double* a_out, double* h_out, int32_t* iters_out, double* residual_out) {
    int64_t m = row_ptr[n];
    int64_t* trp = (int64_t*)malloc((size_t)(n + 1) * sizeof(int64_t));
    int32_t* tcol = (int32_t*)malloc((size_t)(m > 0 ? m : 1) * sizeof(int32_t));
    transpose_pattern(n, row_ptr, col, trp, tcol);
    double* a = (double*)malloc((size_t)n * sizeof(double));
    double* h = (double*)malloc((size_t)n * sizeof(double));
    double* an = (double*)malloc((size_t)n * sizeof(double));
    double* hn = (double*)malloc((size_t)n * sizeof(double));
    for (int64_t i = 0; i < n; ++i) { a[i] = 1.0 / (double)n; h[i] = 1.0 / (double)n; }
    int32_t it = 0; double res = INFINITY; int rc = 1;
    int32_t limit = fixed_iters > 0 ? fixed_iters : max_iter;
    while (it < limit) {
        spmv_d(n, trp, tcol, h, an);     /* a' = A^T h */
        spmv_d(n, row_ptr, col, a, hn);  /* h' = A a   */
        normalise(n, an, norm);
        normalise(n, hn, norm);
        res = l1diff(n, an, a) + l1diff(n, hn, h);
        memcpy(a, an, (size_t)n * sizeof(double));
        memcpy(h, hn, (size_t)n * sizeof(double));
        ++it;
        if (fixed_iters <= 0 && res < tol) { rc = 0; break; }
    }
    if (fixed_iters > 0) rc = 0;
    memcpy(a_out, a, (size_t)n * sizeof(double));
    memcpy(h_out, h, (size_t)n * sizeof(double));
    *iters_out = it; *residual_out = res;
    free(trp); free(tcol); free(a); free(h); free(an); free(hn);
    return rc;
}

static int cmp_i32(const void* x, const void* y) {
    int32_t a = *(const int32_t*)x, b = *(const int32_t*)y; return (a > b) - (a < b);
}

/* RWR, Eq. 9: r' = c W r + (1-c) e_q.  The graph is treated as undirected:
 * S = binary(A u A^T) (duplicates merged, no self loop added), W = S D^-1 with D = diag(deg),
 * i.e. (W r)_i = sum_{j in N(i)} r_j / deg(j).  r(0) = e_q. */
OR_EXPORT int oracle_rwr(int64_t n, const int64_t* row_ptr, const int32_t* col, int64_t query,
                         double c, double tol, int32_t max_iter, int32_t fixed_iters,
                         double* r_out, int32_t* iters_out, double* residual_out) {
    int64_t m = row_ptr[n];
    int64_t* trp = (int64_t*)malloc((size_t)(n + 1) * sizeof(int64_t));
    int32_t* tcol = (int32_t*)malloc((size_t)(m > 0 ? m : 1) * sizeof(int32_t));
    transpose_pattern(n, row_ptr, col, trp, tcol);
    /* S row i = sorted unique union of out-neighbours and in-neighbours of i */
    int64_t* srp = (int64_t*)malloc((size_t)(n + 1) * sizeof(int64_t));
    int32_t* scol = (int32_t*)malloc((size_t)(2 * m > 0 ? 2 * m : 1) * sizeof(int32_t));
    srp[0] = 0;
    int64_t w = 0;
    for (int64_t i = 0; i < n; ++i) {
        int64_t s0 = w;
        for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) scol[w++] = col[k];
        for (int64_t k = trp[i]; k < trp[i + 1]; ++k) scol[w++] = tcol[k];
        qsort(scol + s0, (size_t)(w - s0), sizeof(int32_t), cmp_i32);
        int64_t u = s0;
        for (int64_t k = s0; k < w; ++k)
            if (k == s0 || scol[k] != scol[u - 1]) scol[u++] = scol[k];
        w = u;
        srp[i + 1] = w;
    }
    double* r = (double*)malloc((size_t)n * sizeof(double));
    double* z = (double*)malloc((size_t)n * sizeof(double));
    double* y = (double*)malloc((size_t)n * sizeof(double));
    double* rn = (double*)malloc((size_t)n * sizeof(double));
    for (int64_t i = 0; i < n; ++i) r[i] = (i == query) ? 1.0 : 0.0;
    int32_t it = 0; double res = INFINITY; int rc = 1;
    int32_t limit = fixed_iters > 0 ? fixed_iters : max_iter;
    while (it < limit) {
        for (int64_t j = 0; j < n; ++j) {
            int64_t d = srp[j + 1] - srp[j];
            z[j] = d ? r[j] / (double)d : 0.0;
        }
        spmv_d(n, srp, scol, z, y);                 /* y = W r */
        for (int64_t i = 0; i < n; ++i) rn[i] = c * y[i] + ((i == query) ? (1.0 - c) : 0.0);
        res = l1diff(n, rn, r);
        memcpy(r, rn, (size_t)n * sizeof(double));
        ++it;
        if (fixed_iters <= 0 && res < tol) { rc = 0; break; }
    }
    if (fixed_iters > 0) rc = 0;
    memcpy(r_out, r, (size_t)n * sizeof(double));
    *iters_out = it; *residual_out = res;
    free(trp); free(tcol); free(srp); free(scol); free(r); free(z); free(y); free(rn);
    return rc;
}
