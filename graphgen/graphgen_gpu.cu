/* graphgen_gpu.cu -- the seeded R-MAT generator of graphgen.c, run on the device.
 *
 * Input infrastructure only (like graphgen.c): it draws graphs, it holds none of the method's
 * arithmetic.  It exists for the configurations whose edge lists do not fit the host's memory or
 * patience (c4 it-2004-shaped, 1.15 B edges; c5 uk-union-shaped, 5.5 B edges) and
 * for ranks that each need their own rows of such a graph (SURVEY 8(b) "*_local").
 *
 * Bit-identical to gg_rmat (graphgen.c): the same counter-based draws (splitmix64 of
 * (seed, attempt * scale + level)), the same adaptive rounds (attempt counts computed on the host
 * from the same doubles), the same set semantics (sort + unique), the same thinning (the m smallest
 * hashes of the unique keys; the hash is a bijection of the key, so there are no ties) and the same
 * seeded relabel (order of (hash >> idb << idb | id)).  tests/test_gpu_graphgen.py compares the keys
 * with graphgen.c's on c1, t_mid and c2.
 *
 * Besides the keys: degree counts and the columns of one rank's rows of the iteration matrix
 * (A rows, A^T rows or the HITS block [[0, A^T], [A, 0]]), so a rank's local input never needs
 * the whole edge list on the host.
 */
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/block/block_scan.cuh>
#include <cub/block/block_reduce.cuh>
#include <cuda_runtime.h>

#define GG_EXPORT extern "C" __attribute__((visibility("default")))

static char g_err[512];
GG_EXPORT const char* ggg_last_error(void) { return g_err; }

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
    snprintf(g_err, sizeof g_err, "%s: %s (%s:%d)", #x, cudaGetErrorString(e_), __FILE__, __LINE__); \
    return 10; } } while (0)

__host__ __device__ static inline uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
// gg_draw(seed, k) = mix64(mix64(seed) ^ k * C): S = mix64(seed) precomputed on the host
__device__ static inline uint64_t draw_s(uint64_t S, uint64_t k) { return mix64(S ^ (k * 0xD1B54A32D192ED03ull)); }
__device__ static inline double u01_53(uint64_t r) { return (double)(r >> 11) * (1.0 / 9007199254740992.0); }

static int bits_for(uint64_t n) { int b = 0; while (b < 64 && (1ull << b) < n) ++b; return b; }

/* ---------------------------------------------------------------- R-MAT attempts [k0, k0 + cnt) */
struct RmatP { int scale; double a, ab, abc; uint64_t S; int64_t n; };

__global__ void rmat_draw(RmatP P, uint64_t k0, uint64_t cnt, uint64_t* out, unsigned long long* nout) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i - threadIdx.x < cnt; i += stride) {
        bool ok = false;
        uint64_t key = 0;
        if (i < cnt) {
            const uint64_t k = k0 + i;
            uint64_t uu = 0, vv = 0;
            for (int l = 0; l < P.scale; ++l) {
                const double r = u01_53(draw_s(P.S, k * (uint64_t)P.scale + (uint64_t)l));
                int bu, bv;
                if (r < P.a) { bu = 0; bv = 0; }
                else if (r < P.ab) { bu = 0; bv = 1; }
                else if (r < P.abc) { bu = 1; bv = 0; }
                else { bu = 1; bv = 1; }
                uu = (uu << 1) | (uint64_t)bu; vv = (vv << 1) | (uint64_t)bv;
            }
            ok = uu < (uint64_t)P.n && vv < (uint64_t)P.n && uu != vv;
            key = (uu << 32) | vv;
        }
        // warp-aggregated append (order is irrelevant: the keys are sorted next)
        const unsigned mask = __ballot_sync(0xffffffffu, ok);
        if (!mask) continue;
        const int lane = threadIdx.x & 31;
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(nout, (unsigned long long)__popc(mask));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (ok) out[base + __popc(mask & ((1u << lane) - 1))] = key;
    }
}

/* ---------------------------------------------------------------- stable compaction
 * out[j] = f(in[i]) for the i with pred(in[i], i), in input order.  Two passes over tiles of
 * kTile items: per-tile counts, a scan of the counts, then per-tile block scans and writes. */
constexpr int kThreads = 256, kPer = 16, kTile = kThreads * kPer;

template <class Pred>
__global__ void tile_count(const uint64_t* in, int64_t n, Pred pred, int64_t* counts) {
    const int64_t t0 = (int64_t)blockIdx.x * kTile;
    int c = 0;
    for (int j = 0; j < kPer; ++j) {
        const int64_t i = t0 + (int64_t)j * kThreads + threadIdx.x;
        if (i < n && pred(in[i], i)) ++c;
    }
    typedef cub::BlockReduce<int, kThreads> BR;
    __shared__ typename BR::TempStorage tmp;
    const int tot = BR(tmp).Sum(c);
    if (threadIdx.x == 0) counts[blockIdx.x] = tot;
}

template <class Pred, class Xf, class OutT>
__global__ void tile_write(const uint64_t* in, int64_t n, Pred pred, Xf xf, const int64_t* offs, OutT* out) {
    const int64_t t0 = (int64_t)blockIdx.x * kTile;
    // thread t handles the contiguous run [t0 + t*kPer, +kPer) so the output keeps input order
    uint64_t v[kPer];
    bool f[kPer];
    int c = 0;
    for (int j = 0; j < kPer; ++j) {
        const int64_t i = t0 + (int64_t)threadIdx.x * kPer + j;
        f[j] = false;
        if (i < n) { v[j] = in[i]; f[j] = pred(v[j], i); c += f[j]; }
    }
    typedef cub::BlockScan<int, kThreads> BS;
    __shared__ typename BS::TempStorage tmp;
    int pre;
    BS(tmp).ExclusiveSum(c, pre);
    int64_t o = offs[blockIdx.x] + pre;
    for (int j = 0; j < kPer; ++j)
        if (f[j]) out[o++] = xf(v[j]);
}

struct Scratch {
    void* p = nullptr; size_t bytes = 0;
    int need(size_t b) {
        if (b <= bytes) return 0;
        if (p) cudaFree(p);
        p = nullptr; bytes = 0;
        if (cudaMalloc(&p, b) != cudaSuccess) return 1;
        bytes = b;
        return 0;
    }
    ~Scratch() { if (p) cudaFree(p); }
};

template <class Pred, class Xf, class OutT>
static int compact(const uint64_t* in, int64_t n, Pred pred, Xf xf, OutT* out, int64_t* n_out, Scratch& sc) {
    *n_out = 0;
    if (n == 0) return 0;
    const int64_t tiles = (n + kTile - 1) / kTile;
    int64_t* cnt = nullptr;
    CK(cudaMalloc(&cnt, (tiles + 1) * sizeof(int64_t)));
    tile_count<<<(unsigned)tiles, kThreads>>>(in, n, pred, cnt);
    CK(cudaGetLastError());
    CK(cudaMemset(cnt + tiles, 0, sizeof(int64_t)));
    size_t tb = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, cnt, tiles + 1));
    if (sc.need(tb)) { cudaFree(cnt); snprintf(g_err, sizeof g_err, "scan scratch"); return 11; }
    CK(cub::DeviceScan::ExclusiveSum(sc.p, tb, cnt, cnt, tiles + 1));
    tile_write<<<(unsigned)tiles, kThreads>>>(in, n, pred, xf, cnt, out);
    CK(cudaGetLastError());
    CK(cudaMemcpy(n_out, cnt + tiles, sizeof(int64_t), cudaMemcpyDeviceToHost));
    CK(cudaFree(cnt));
    return 0;
}

// sort keys[0, n) (bits [0, end_bit)); the result lands in *cur (one of a / b)
static int sort_keys(uint64_t*& a, uint64_t*& b, int64_t n, int end_bit, Scratch& sc) {
    if (n <= 1) return 0;
    cub::DoubleBuffer<uint64_t> db(a, b);
    size_t tb = 0;
    CK(cub::DeviceRadixSort::SortKeys(nullptr, tb, db, n, 0, end_bit));
    if (sc.need(tb)) { snprintf(g_err, sizeof g_err, "sort scratch (%zu bytes)", tb); return 11; }
    CK(cub::DeviceRadixSort::SortKeys(sc.p, tb, db, n, 0, end_bit));
    if (db.Current() != a) { uint64_t* t = a; a = b; b = t; }
    return 0;
}

struct PredUnique {
    const uint64_t* k;
    __device__ bool operator()(uint64_t v, int64_t i) const { return i == 0 || k[i - 1] != v; }
};
struct Ident { __device__ uint64_t operator()(uint64_t v) const { return v; } };

/* ---------------------------------------------------------------- thinning: the (m-1)-th smallest hash */
__global__ void hash_hist(const uint64_t* keys, int64_t n, uint64_t S, int shift, uint64_t prefix, uint64_t pmask,
                          unsigned long long* hist) {
    __shared__ unsigned int h[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t hv = draw_s(S, keys[i]);
        if ((hv & pmask) == prefix) atomicAdd(&h[(hv >> shift) & 255], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 256; i += blockDim.x)
        if (h[i]) atomicAdd(&hist[i], (unsigned long long)h[i]);
}
struct PredHashLe {
    uint64_t S, thr;
    __device__ bool operator()(uint64_t v, int64_t) const { return draw_s(S, v) <= thr; }
};

/* ---------------------------------------------------------------- relabel */
__global__ void relabel_keys(uint64_t S, int idb, int64_t n, uint64_t* k) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        k[i] = ((draw_s(S, (uint64_t)i) >> idb) << idb) | (uint64_t)i;
}
__global__ void relabel_scatter(const uint64_t* k, int64_t n, uint64_t mask, int32_t* lab) {
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x)
        lab[k[p] & mask] = (int32_t)p;
}
__global__ void apply_relabel(const uint64_t* in, int64_t m, const int32_t* lab, uint64_t* out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t u = in[i] >> 32, v = in[i] & 0xFFFFFFFFull;
        out[i] = ((uint64_t)(uint32_t)lab[u] << 32) | (uint64_t)(uint32_t)lab[v];
    }
}

static unsigned grid_for(int64_t n) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t g = (n + 255) / 256;
    if (g > (int64_t)sms * 16) g = (int64_t)sms * 16;
    return (unsigned)(g < 1 ? 1 : g);
}

/* gg_rmat on the device: *d_keys_out = device buffer (free with ggg_free) of the *m_out sorted
 * unique keys (u << 32) | v.  Returns 0, 1 (bad arguments), 2 (no convergence), >= 10 (CUDA). */
GG_EXPORT int ggg_rmat(int scale, int64_t n, int64_t m, double a, double b, double c, uint64_t seed,
                       uint64_t relabel_seed, int device, uint64_t** d_keys_out, int64_t* m_out) {
    g_err[0] = 0;
    if (scale < 1 || scale > 31 || n > (1ll << scale) || n < 2 || m < 0 || (double)m > (double)n * (double)(n - 1))
        return 1;
    CK(cudaSetDevice(device));
    RmatP P{scale, a, a + b, a + b + c, mix64(seed), n};
    int64_t cap = m + m / 4 + 1024, have = 0;
    uint64_t *A = nullptr, *B = nullptr;
    CK(cudaMalloc(&A, (size_t)cap * 8));
    if (cudaMalloc(&B, (size_t)cap * 8) != cudaSuccess) { cudaFree(A); snprintf(g_err, sizeof g_err, "key buffers"); return 12; }
    Scratch sc;
    unsigned long long* d_n = nullptr;
    int rc = 0;
    const int key_bits = 32 + bits_for((uint64_t)n);
    auto fail = [&](int r) { cudaFree(A); cudaFree(B); if (d_n) cudaFree(d_n); return r; };
    if (cudaMalloc(&d_n, sizeof(unsigned long long)) != cudaSuccess) return fail(12);
    uint64_t k = 0;
    double accept = 1.0;
    int rounds = 0;
    while (have < m) {
        const int64_t need = m - have;
        uint64_t attempts = (uint64_t)((double)need / accept * 1.05) + 1024;
        if ((int64_t)attempts > 4 * cap) attempts = (uint64_t)(4 * cap);
        const int64_t room = have + (int64_t)attempts;
        if (room > cap) {   // graphgen.c reallocs; here: grow both buffers, keep the keys
            uint64_t *A2 = nullptr, *B2 = nullptr;
            if (cudaMalloc(&A2, (size_t)room * 8) != cudaSuccess) return fail(12);
            cudaMemcpy(A2, A, (size_t)have * 8, cudaMemcpyDeviceToDevice);
            cudaFree(A); A = A2;
            cudaFree(B);
            if (cudaMalloc(&B2, (size_t)room * 8) != cudaSuccess) { B = nullptr; return fail(12); }
            B = B2; cap = room;
        }
        cudaMemset(d_n, 0, sizeof(unsigned long long));
        rmat_draw<<<grid_for((int64_t)attempts) * 2, 256>>>(P, k, attempts, A + have, d_n);
        if (cudaGetLastError() != cudaSuccess) return fail(13);
        unsigned long long got = 0;
        if (cudaMemcpy(&got, d_n, sizeof got, cudaMemcpyDeviceToHost) != cudaSuccess) return fail(13);
        const int64_t before = have;
        if ((rc = sort_keys(A, B, have + (int64_t)got, key_bits, sc))) return fail(rc);
        int64_t u = 0;
        if ((rc = compact(A, have + (int64_t)got, PredUnique{A}, Ident{}, B, &u, sc))) return fail(rc);
        { uint64_t* t = A; A = B; B = t; }
        have = u;
        k += attempts;
        const double acc = (double)(have - before) / (double)attempts;
        if (acc > 1e-6) accept = acc; else accept *= 0.5;
        if (++rounds > 200) return fail(2);
    }
    // thin_to(keys, have, m, seed ^ 0x7417A11): keep the m smallest hashes (distinct: a bijection)
    if (have > m) {
        const uint64_t Sth = mix64(seed ^ 0x7417A11ull);
        unsigned long long* hist = nullptr;
        if (cudaMalloc(&hist, 256 * sizeof(unsigned long long)) != cudaSuccess) return fail(12);
        uint64_t prefix = 0, pmask = 0;
        int64_t kk = m - 1;                 // rank among the keys matching the prefix
        for (int shift = 56; shift >= 0; shift -= 8) {
            cudaMemset(hist, 0, 256 * sizeof(unsigned long long));
            hash_hist<<<grid_for(have), 256>>>(A, have, Sth, shift, prefix, pmask, hist);
            unsigned long long h[256];
            if (cudaMemcpy(h, hist, sizeof h, cudaMemcpyDeviceToHost) != cudaSuccess) { cudaFree(hist); return fail(13); }
            int d = 0;
            while (d < 255 && (int64_t)h[d] <= kk) { kk -= (int64_t)h[d]; ++d; }
            prefix |= (uint64_t)d << shift;
            pmask |= 255ull << shift;
        }
        cudaFree(hist);
        int64_t w = 0;
        if ((rc = compact(A, have, PredHashLe{Sth, prefix}, Ident{}, B, &w, sc))) return fail(rc);
        { uint64_t* t = A; A = B; B = t; }
        if (w != m) { snprintf(g_err, sizeof g_err, "thinning kept %lld of %lld", (long long)w, (long long)m); return fail(14); }
        have = w;
    }
    if (relabel_seed != 0) {
        int idb = bits_for((uint64_t)n); if (idb < 1) idb = 1;
        const uint64_t mask = (idb >= 64) ? ~0ull : ((1ull << idb) - 1);
        uint64_t *R = nullptr, *R2 = nullptr;
        int32_t* lab = nullptr;
        if (cudaMalloc(&R, (size_t)n * 8) || cudaMalloc(&R2, (size_t)n * 8) || cudaMalloc(&lab, (size_t)n * 4)) {
            cudaFree(R); cudaFree(R2); cudaFree(lab); return fail(12);
        }
        relabel_keys<<<grid_for(n), 256>>>(mix64(relabel_seed), idb, n, R);
        if ((rc = sort_keys(R, R2, n, 64, sc))) { cudaFree(R); cudaFree(R2); cudaFree(lab); return fail(rc); }
        relabel_scatter<<<grid_for(n), 256>>>(R, n, mask, lab);
        apply_relabel<<<grid_for(have), 256>>>(A, have, lab, B);
        cudaFree(R); cudaFree(R2); cudaFree(lab);
        { uint64_t* t = A; A = B; B = t; }
        if ((rc = sort_keys(A, B, have, 32 + idb, sc))) return fail(rc);
    }
    if (cudaDeviceSynchronize() != cudaSuccess) return fail(13);
    cudaFree(B);
    cudaFree(d_n);
    *d_keys_out = A;
    *m_out = have;
    return 0;
}

GG_EXPORT void ggg_free(void* d) { if (d) cudaFree(d); }

GG_EXPORT int ggg_to_host(const uint64_t* d_keys, int64_t m, uint64_t* h_out) {
    CK(cudaMemcpy(h_out, d_keys, (size_t)m * 8, cudaMemcpyDeviceToHost));
    return 0;
}

/* ---------------------------------------------------------------- degrees */
__global__ void degree_count(const uint64_t* keys, int64_t m, int32_t* out_deg, int32_t* in_deg) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t k = keys[i];
        atomicAdd(&out_deg[k >> 32], 1);
        atomicAdd(&in_deg[k & 0xFFFFFFFFull], 1);
    }
}

/* out-degree (key >> 32) and in-degree (key & 0xffffffff) of every vertex, to host int32 [n]. */
GG_EXPORT int ggg_degrees(const uint64_t* d_keys, int64_t m, int64_t n, int32_t* h_out_deg, int32_t* h_in_deg) {
    g_err[0] = 0;
    int32_t* d = nullptr;
    CK(cudaMalloc(&d, (size_t)2 * n * 4));
    CK(cudaMemset(d, 0, (size_t)2 * n * 4));
    degree_count<<<grid_for(m), 256>>>(d_keys, m, d, d + n);
    CK(cudaGetLastError());
    CK(cudaMemcpy(h_out_deg, d, (size_t)n * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(h_in_deg, d + n, (size_t)n * 4, cudaMemcpyDeviceToHost));
    CK(cudaFree(d));
    return 0;
}

/* ---------------------------------------------------------------- one rank's rows */
struct PredOwner {     // owner of the row the key falls in: row = key >> 32 (+ off) or the low half (+ off)
    const int32_t* owner; int hi; int64_t off; int32_t q;
    __device__ bool operator()(uint64_t v, int64_t) const {
        const int64_t r = (int64_t)(hi ? (v >> 32) : (v & 0xFFFFFFFFull)) + off;
        return owner[r] == q;
    }
};
struct Swap { __device__ uint64_t operator()(uint64_t v) const { return (v << 32) | (v >> 32); } };
__global__ void low_plus(const uint64_t* in, int64_t cnt, int64_t add, int32_t* out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (int32_t)((int64_t)(in[i] & 0xFFFFFFFFull) + add);
}

/* The column ids of rank q's rows of an iteration matrix built from the keys, rows in ascending
 * id, each row's columns ascending (the host derives the row ids and row_ptr from the owner array
 * and the degrees):
 *   kind 0: A      (row u lists v; N = n)
 *   kind 1: A^T    (row v lists u; N = n)       -- PageRank's iteration matrix (Eq. 6)
 *   kind 2: [[0, A^T], [A, 0]] (N = 2n: row v < n lists n + u, row n + u lists v) -- HITS (Eq. 8)
 * h_owner: int32 [N] on the host.  *h_col_out: malloc'ed host int32 [*cnt_out] (free with ggg_host_free). */
GG_EXPORT int ggg_owned_cols(const uint64_t* d_keys, int64_t m, int64_t n, int kind, const int32_t* h_owner,
                             int32_t q, int32_t** h_col_out, int64_t* cnt_out) {
    g_err[0] = 0;
    if (kind < 0 || kind > 2) return 1;
    const int64_t N = kind == 2 ? 2 * n : n;
    int32_t* d_owner = nullptr;
    CK(cudaMalloc(&d_owner, (size_t)N * 4));
    CK(cudaMemcpy(d_owner, h_owner, (size_t)N * 4, cudaMemcpyHostToDevice));
    Scratch sc;
    std::vector<int32_t*> parts;     // device int32 columns, in output order
    std::vector<int64_t> counts;
    const int idb = bits_for((uint64_t)n) < 1 ? 1 : bits_for((uint64_t)n);
    auto take = [&](int transposed, int64_t col_add, int64_t row_off) -> int {
        // transposed: row = low half (v), select then swap to (v, u) and sort; else row = high half
        uint64_t *E = nullptr, *E2 = nullptr;
        int64_t c = 0;
        // count first to size the buffers
        {
            int64_t* tmp = nullptr;
            const int64_t tiles = (m + kTile - 1) / kTile;
            CK(cudaMalloc(&tmp, (tiles + 1) * sizeof(int64_t)));
            if (m) tile_count<<<(unsigned)tiles, kThreads>>>(d_keys, m, PredOwner{d_owner, !transposed, row_off, q}, tmp);
            std::vector<int64_t> h(tiles);
            CK(cudaMemcpy(h.data(), tmp, tiles * sizeof(int64_t), cudaMemcpyDeviceToHost));
            cudaFree(tmp);
            for (int64_t t = 0; t < tiles; ++t) c += h[t];
        }
        int32_t* out = nullptr;
        CK(cudaMalloc(&E, (size_t)(c + 1) * 8));
        int64_t w = 0;
        int rc;
        if (transposed) {
            if ((rc = compact(d_keys, m, PredOwner{d_owner, 0, row_off, q}, Swap{}, E, &w, sc))) { cudaFree(E); return rc; }
            CK(cudaMalloc(&E2, (size_t)(c + 1) * 8));
            if ((rc = sort_keys(E, E2, w, 32 + idb, sc))) { cudaFree(E); cudaFree(E2); return rc; }
            cudaFree(E2);
        } else {
            if ((rc = compact(d_keys, m, PredOwner{d_owner, 1, row_off, q}, Ident{}, E, &w, sc))) { cudaFree(E); return rc; }
        }
        CK(cudaMalloc(&out, (size_t)(w + 1) * 4));
        if (w) low_plus<<<grid_for(w), 256>>>(E, w, col_add, out);
        CK(cudaGetLastError());
        cudaFree(E);
        parts.push_back(out); counts.push_back(w);
        return 0;
    };
    int rc = 0;
    if (kind == 0) rc = take(0, 0, 0);
    else if (kind == 1) rc = take(1, 0, 0);
    else {
        rc = take(1, n, 0);          // rows v < n of A^T: columns n + u
        if (!rc) rc = take(0, 0, n); // rows n + u of A: columns v
    }
    cudaFree(d_owner);
    if (rc) { for (auto p : parts) cudaFree(p); return rc; }
    int64_t tot = 0;
    for (int64_t c : counts) tot += c;
    int32_t* h = (int32_t*)malloc((size_t)(tot + 1) * 4);
    if (!h) { for (auto p : parts) cudaFree(p); snprintf(g_err, sizeof g_err, "host allocation"); return 12; }
    int64_t o = 0;
    for (size_t i = 0; i < parts.size(); ++i) {
        if (counts[i]) CK(cudaMemcpy(h + o, parts[i], (size_t)counts[i] * 4, cudaMemcpyDeviceToHost));
        o += counts[i];
        cudaFree(parts[i]);
    }
    *h_col_out = h;
    *cnt_out = tot;
    return 0;
}

GG_EXPORT void ggg_host_free(void* p) { free(p); }
