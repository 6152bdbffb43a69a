/*
 * graphgen.c -- seeded synthetic inputs shared by the oracle and the product path.
 *
 * This module holds NONE of the method's arithmetic (no SpMV, no reordering, no tiling,
 * no packing, no power iteration).  It only draws inputs:
 *   - R-MAT / Kronecker directed graphs (Chakrabarti et al.; Graph500 parameters), used as
 *     stand-ins for the paper's power-law graphs (Table 2, L307-L313 Table 3),
 *   - capped Chung-Lu power-law graphs for the skew sweep,
 *   - counter-based uniform fp32 vectors (x, matrix values).
 *
 * Every random number is a pure function of (seed, counter) through splitmix64, so any
 * consumer (oracle, GPU path, a rank that regenerates its rows) gets the same bits.
 * Output edges are unique, have no self loops and are returned as sorted 64-bit keys
 * key = (u << 32) | v  for the directed edge u -> v (A(u,v) = 1).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define GG_EXPORT __attribute__((visibility("default")))

static inline uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* counter-based generator: the k-th 64-bit draw of stream `seed` */
GG_EXPORT uint64_t gg_draw(uint64_t seed, uint64_t k) {
    return mix64(mix64(seed) ^ (k * 0xD1B54A32D192ED03ull));
}

static inline double u01_53(uint64_t r) { return (double)(r >> 11) * (1.0 / 9007199254740992.0); }

/* ---------------------------------------------------------------- radix sort (u64) */
static void radix_sort_u64(uint64_t* a, int64_t n, int key_bits) {
    if (n <= 1) return;
    uint64_t* tmp = (uint64_t*)malloc((size_t)n * sizeof(uint64_t));
    uint64_t* src = a; uint64_t* dst = tmp;
    int passes = (key_bits + 15) / 16;
    for (int p = 0; p < passes; ++p) {
        int shift = 16 * p;
        int64_t* cnt = (int64_t*)calloc(65537, sizeof(int64_t));
        for (int64_t i = 0; i < n; ++i) cnt[((src[i] >> shift) & 0xFFFF) + 1]++;
        for (int d = 0; d < 65536; ++d) cnt[d + 1] += cnt[d];
        for (int64_t i = 0; i < n; ++i) dst[cnt[(src[i] >> shift) & 0xFFFF]++] = src[i];
        free(cnt);
        uint64_t* t = src; src = dst; dst = t;
    }
    if (src != a) memcpy(a, src, (size_t)n * sizeof(uint64_t));
    free(tmp);
}

static int64_t unique_sorted(uint64_t* a, int64_t n) {
    if (n == 0) return 0;
    int64_t w = 1;
    for (int64_t i = 1; i < n; ++i) if (a[i] != a[w - 1]) a[w++] = a[i];
    return w;
}

static int bits_for(uint64_t n) { int b = 0; while (b < 64 && (1ull << b) < n) ++b; return b; }

/* random permutation of [0,n): new label of vertex i = position of i when ids are ordered by
 * (hash(seed, i) top bits, i).  Returns malloc'ed int64 array newlabel[i]. */
static int64_t* random_relabel(int64_t n, uint64_t seed) {
    int idb = bits_for((uint64_t)n); if (idb < 1) idb = 1;
    uint64_t* k = (uint64_t*)malloc((size_t)n * sizeof(uint64_t));
    uint64_t mask = (idb >= 64) ? ~0ull : ((1ull << idb) - 1);
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) k[i] = ((gg_draw(seed, (uint64_t)i) >> idb) << idb) | (uint64_t)i;
    radix_sort_u64(k, n, 64);
    int64_t* lab = (int64_t*)malloc((size_t)n * sizeof(int64_t));
    for (int64_t p = 0; p < n; ++p) lab[k[p] & mask] = p;
    free(k);
    return lab;
}

/* keep exactly m of the n (sorted, unique) keys: the m smallest by hash(seed, key) */
static int cmp_u64(const void* x, const void* y) {
    uint64_t a = *(const uint64_t*)x, b = *(const uint64_t*)y; return (a > b) - (a < b);
}
static uint64_t kth_smallest(uint64_t* v, int64_t n, int64_t k) {
    int64_t lo = 0, hi = n - 1;
    while (hi - lo > 16) {
        uint64_t piv = v[lo + (hi - lo) / 2];
        int64_t i = lo, j = hi;
        while (i <= j) {
            while (v[i] < piv) ++i;
            while (v[j] > piv) --j;
            if (i <= j) { uint64_t t = v[i]; v[i] = v[j]; v[j] = t; ++i; --j; }
        }
        if (k <= j) hi = j; else if (k >= i) lo = i; else return v[k];
    }
    qsort(v + lo, (size_t)(hi - lo + 1), sizeof(uint64_t), cmp_u64);
    return v[k];
}
static int64_t thin_to(uint64_t* keys, int64_t n, int64_t m, uint64_t seed) {
    if (n <= m) return n;
    uint64_t* h = (uint64_t*)malloc((size_t)n * sizeof(uint64_t));
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) h[i] = gg_draw(seed, keys[i]);
    uint64_t* hc = (uint64_t*)malloc((size_t)n * sizeof(uint64_t));
    memcpy(hc, h, (size_t)n * sizeof(uint64_t));
    uint64_t thr = kth_smallest(hc, n, m - 1);
    free(hc);
    int64_t below = 0;
    for (int64_t i = 0; i < n; ++i) below += (h[i] < thr);
    int64_t eq_keep = m - below, w = 0;
    for (int64_t i = 0; i < n; ++i) {
        if (h[i] < thr) keys[w++] = keys[i];
        else if (h[i] == thr && eq_keep > 0) { keys[w++] = keys[i]; --eq_keep; }
    }
    free(h);
    return w;
}

/* ---------------------------------------------------------------- edge samplers */
typedef int (*edge_fn)(const void* ctx, uint64_t k, uint64_t* u, uint64_t* v);

typedef struct { int scale; double a, ab, abc; uint64_t seed; } rmat_ctx;
static int rmat_edge(const void* c_, uint64_t k, uint64_t* u, uint64_t* v) {
    const rmat_ctx* c = (const rmat_ctx*)c_;
    uint64_t uu = 0, vv = 0;
    for (int l = 0; l < c->scale; ++l) {
        double r = u01_53(gg_draw(c->seed, k * (uint64_t)c->scale + (uint64_t)l));
        int bu, bv;
        if (r < c->a) { bu = 0; bv = 0; }
        else if (r < c->ab) { bu = 0; bv = 1; }
        else if (r < c->abc) { bu = 1; bv = 0; }
        else { bu = 1; bv = 1; }
        uu = (uu << 1) | (uint64_t)bu; vv = (vv << 1) | (uint64_t)bv;
    }
    *u = uu; *v = vv;
    return 1;
}

typedef struct { int64_t n; const double* cdf; uint64_t seed; } cl_ctx;
static int64_t cdf_pick(const double* cdf, int64_t n, double r) {
    int64_t lo = 0, hi = n - 1;   /* first i with cdf[i] > r */
    while (lo < hi) { int64_t mid = (lo + hi) >> 1; if (cdf[mid] > r) hi = mid; else lo = mid + 1; }
    return lo;
}
static int cl_edge(const void* c_, uint64_t k, uint64_t* u, uint64_t* v) {
    const cl_ctx* c = (const cl_ctx*)c_;
    *u = (uint64_t)cdf_pick(c->cdf, c->n, u01_53(gg_draw(c->seed, 2 * k)));
    *v = (uint64_t)cdf_pick(c->cdf, c->n, u01_53(gg_draw(c->seed, 2 * k + 1)));
    return 1;
}

/* draw attempts [k0,k1), keep edges with u,v < n and u != v; returns count appended */
static int64_t draw_range(edge_fn f, const void* ctx, int64_t n, uint64_t k0, uint64_t k1,
                          uint64_t* out) {
    int nt = 1;
#ifdef _OPENMP
    nt = omp_get_max_threads();
#endif
    int64_t total = (int64_t)(k1 - k0);
    int64_t* cnt = (int64_t*)calloc((size_t)nt + 1, sizeof(int64_t));
    uint64_t** bufs = (uint64_t**)calloc((size_t)nt, sizeof(uint64_t*));
    #pragma omp parallel num_threads(nt)
    {
        int t = 0;
#ifdef _OPENMP
        t = omp_get_thread_num();
#endif
        int64_t lo = total * t / nt, hi = total * (t + 1) / nt;
        uint64_t* b = (uint64_t*)malloc((size_t)(hi - lo + 1) * sizeof(uint64_t));
        int64_t c = 0;
        for (int64_t i = lo; i < hi; ++i) {
            uint64_t u, v;
            f(ctx, k0 + (uint64_t)i, &u, &v);
            if (u >= (uint64_t)n || v >= (uint64_t)n || u == v) continue;
            b[c++] = (u << 32) | v;
        }
        bufs[t] = b; cnt[t] = c;
    }
    int64_t w = 0;
    for (int t = 0; t < nt; ++t) { memcpy(out + w, bufs[t], (size_t)cnt[t] * sizeof(uint64_t)); w += cnt[t]; free(bufs[t]); }
    free(bufs); free(cnt);
    return w;
}

/* generic: draw until >= m unique edges, thin to m, relabel, sort. */
static int gen_edges(edge_fn f, const void* ctx, int64_t n, int64_t m, uint64_t seed,
                     uint64_t relabel_seed, uint64_t** keys_out, int64_t* m_out) {
    if (n < 2 || m < 0 || (double)m > (double)n * (double)(n - 1)) return 1;
    int64_t cap = m + m / 4 + 1024, have = 0;
    uint64_t* keys = (uint64_t*)malloc((size_t)cap * sizeof(uint64_t));
    uint64_t k = 0;
    double accept = 1.0;          /* unique edges per attempt, refined as we go */
    int rounds = 0;
    while (have < m) {
        int64_t need = m - have;
        uint64_t attempts = (uint64_t)((double)need / accept * 1.05) + 1024;
        if ((int64_t)attempts > 4 * cap) attempts = (uint64_t)(4 * cap);
        int64_t room = have + (int64_t)attempts;
        if (room > cap) { cap = room; keys = (uint64_t*)realloc(keys, (size_t)cap * sizeof(uint64_t)); }
        int64_t got = draw_range(f, ctx, n, k, k + attempts, keys + have);
        int64_t before = have;
        radix_sort_u64(keys, have + got, 64);
        have = unique_sorted(keys, have + got);
        k += attempts;
        double acc = (double)(have - before) / (double)attempts;
        if (acc > 1e-6) accept = acc; else accept *= 0.5;
        if (++rounds > 200) { free(keys); return 2; }
    }
    have = thin_to(keys, have, m, seed ^ 0x7417A11ull);
    if (relabel_seed != 0) {
        int64_t* lab = random_relabel(n, relabel_seed);
        #pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < have; ++i) {
            uint64_t u = keys[i] >> 32, v = keys[i] & 0xFFFFFFFFull;
            keys[i] = ((uint64_t)lab[u] << 32) | (uint64_t)lab[v];
        }
        free(lab);
        radix_sort_u64(keys, have, 64);
    }
    *keys_out = keys; *m_out = have;
    return 0;
}

/* R-MAT over a 2^scale grid, ids >= n rejected; d = 1 - a - b - c. */
GG_EXPORT int gg_rmat(int scale, int64_t n, int64_t m, double a, double b, double c,
                      uint64_t seed, uint64_t relabel_seed, uint64_t** keys_out, int64_t* m_out) {
    if (scale < 1 || scale > 31 || n > (1ll << scale)) return 1;
    rmat_ctx ctx = { scale, a, a + b, a + b + c, seed };
    return gen_edges(rmat_edge, &ctx, n, m, seed, relabel_seed, keys_out, m_out);
}

/* capped Chung-Lu: weight_i = (i + i0)^(-1/(alpha-1)); i0 chosen so that the expected
 * degree (in == out) of vertex 0, m * w_0 / sum(w), equals max_deg. */
GG_EXPORT int gg_chung_lu(int64_t n, int64_t m, double alpha, double max_deg, uint64_t seed,
                          uint64_t relabel_seed, uint64_t** keys_out, int64_t* m_out) {
    if (alpha <= 1.0 || n < 2) return 1;
    double g = 1.0 / (alpha - 1.0);
    double* cdf = (double*)malloc((size_t)n * sizeof(double));
    double lo = 0.0, hi = (double)n * 4.0, i0 = 1.0;
    for (int it = 0; it < 200; ++it) {
        i0 = 0.5 * (lo + hi);
        double s = 0.0;
        for (int64_t i = 0; i < n; ++i) s += pow((double)i + i0, -g);
        double d0 = (double)m * pow(i0, -g) / s;
        if (d0 > max_deg) lo = i0; else hi = i0;   /* larger i0 -> flatter -> smaller d0 */
        if (hi - lo < 1e-9 * (1.0 + i0)) break;
    }
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) { s += pow((double)i + i0, -g); cdf[i] = s; }
    for (int64_t i = 0; i < n; ++i) cdf[i] /= s;
    cdf[n - 1] = 1.0;
    cl_ctx ctx = { n, cdf, seed };
    int rc = gen_edges(cl_edge, &ctx, n, m, seed, relabel_seed, keys_out, m_out);
    free(cdf);
    return rc;
}

/* sorted unique keys -> CSR.  transpose = 0: row u holds targets v (A);  1: row v holds sources u. */
GG_EXPORT void gg_keys_to_csr(const uint64_t* keys, int64_t m, int64_t n, int transpose,
                              int64_t* row_ptr, int32_t* col) {
    memset(row_ptr, 0, (size_t)(n + 1) * sizeof(int64_t));
    for (int64_t i = 0; i < m; ++i) {
        uint64_t r = transpose ? (keys[i] & 0xFFFFFFFFull) : (keys[i] >> 32);
        row_ptr[r + 1]++;
    }
    for (int64_t i = 0; i < n; ++i) row_ptr[i + 1] += row_ptr[i];
    if (!transpose) {
        for (int64_t i = 0; i < m; ++i) col[i] = (int32_t)(keys[i] & 0xFFFFFFFFull);
        return;
    }
    int64_t* pos = (int64_t*)malloc((size_t)n * sizeof(int64_t));
    memcpy(pos, row_ptr, (size_t)n * sizeof(int64_t));
    for (int64_t i = 0; i < m; ++i) {   /* keys sorted by (u,v): rows of A^T get u ascending */
        uint64_t r = keys[i] & 0xFFFFFFFFull;
        col[pos[r]++] = (int32_t)(keys[i] >> 32);
    }
    free(pos);
}

/* fp32 uniforms: out[i] = U[0,1) (open_lo = 0) or U(0,1] (open_lo = 1), 24-bit exact;
 * signed = 1 maps to U(-1,1) (2*u-1 with u in (0,1)). draw index = offset + i. */
GG_EXPORT void gg_uniform_f32(uint64_t seed, uint64_t offset, int64_t count, int mode, float* out) {
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < count; ++i) {
        uint64_t r = gg_draw(seed, offset + (uint64_t)i) >> 40;  /* 24 bits */
        float u;
        if (mode == 0) u = (float)r * (1.0f / 16777216.0f);
        else if (mode == 1) u = (float)(r + 1) * (1.0f / 16777216.0f);
        else u = ((float)(r | 1) * (1.0f / 16777216.0f)) * 2.0f - 1.0f;  /* signed, never 0 */
        out[i] = u;
    }
}

/* per-edge values keyed by the edge key (independent of storage order) */
GG_EXPORT void gg_edge_values_f32(uint64_t seed, const uint64_t* keys, int64_t m, int mode, float* out) {
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < m; ++i) {
        uint64_t r = gg_draw(seed, keys[i]) >> 40;
        float u;
        if (mode == 0) u = (float)r * (1.0f / 16777216.0f);
        else if (mode == 1) u = (float)(r + 1) * (1.0f / 16777216.0f);
        else u = ((float)(r | 1) * (1.0f / 16777216.0f)) * 2.0f - 1.0f;
        out[i] = u;
    }
}

GG_EXPORT void gg_free(void* p) { free(p); }
