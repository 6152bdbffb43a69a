// iterate.cu -- PageRank (Eq. 6), HITS (Eq. 7-8) and RWR (Eq. 9) power iterations on the
// tiled-composite SpMV, with the vector work fused into the SpMV's row writes (SURVEY.md 8(a)
// a11-a14; App. F).
//
// Every graph is relabelled symmetrically by the column length of its iteration matrix (Solution
// 2, L66, applied to rows and columns), so the SpMV output in relabelled space is directly the
// next input: no per-iteration permutation.
//   PageRank: M = A^T (pattern), z = p * inv_outdeg; y = M z = W^T p; the row's final write
//             applies p' = c (y + D/n) + (1-c)/n (dangling mass D redistributed, reading R1),
//             z' = p' inv_outdeg, and fp64 partials of |p' - p| and of the next D.
//   RWR:      M = binary(A u A^T), z = r * inv_deg; r' = c y + (1-c) e_q (Eq. 9, reading R6).
//   HITS:     M = [[0, A^T], [A, 0]] (Eq. 8, 2n rows); the SpMV's final writes accumulate the two
//             half norms; a second pass divides each half by its norm (L440: "two vector division
//             by constant kernels") and accumulates the L1 change.
// Reductions: per-block fp64 partials in fixed slots, summed in a fixed order by the last block
// (deterministic; no atomics on values).  The loop runs on the device: a CUDA graph whose WHILE
// conditional node repeats the iteration until the last block clears the condition.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <vector>

#include "launch.cuh"
#include "solver.h"

namespace tc {

spmv_status create_plan(int64_t n_rows, int64_t n_cols, int64_t nnz, const int64_t* row_ptr,
                        const int32_t* col, const float* val, const spmv_options* opt_in,
                        int device, spmv_plan_s** out);

// ------------------------------------------------------------------ device helpers
template <int NP>
__device__ __forceinline__ void block_reduce_to_slot(double (&v)[NP], double* slot) {
    __shared__ double red[kWarps][NP];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    #pragma unroll
    for (int k = 0; k < NP; ++k)
        for (int o = 16; o >= 1; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
    if (lane == 0) {
        #pragma unroll
        for (int k = 0; k < NP; ++k) red[warp][k] = v[k];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        #pragma unroll
        for (int k = 0; k < NP; ++k) {
            double s = 0.0;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w][k];
            slot[k] = s;
        }
    }
}

// true in exactly one (the last arriving) block of this launch
__device__ __forceinline__ bool last_block(uint32_t* ticket) {
    __shared__ bool am_last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        uint32_t t = atomicAdd(ticket, 1u);
        am_last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (am_last) __threadfence();
    return am_last;
}

// fixed-order sum of slots[0..n)[k] by the whole block; result valid in thread 0
template <int NP>
__device__ __forceinline__ void block_sum_slots(const double* slots, int n, double (&out)[NP]) {
    double v[NP];
    #pragma unroll
    for (int k = 0; k < NP; ++k) v[k] = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        #pragma unroll
        for (int k = 0; k < NP; ++k) v[k] += __ldcg(slots + (size_t)i * NP + k);
    }
    __shared__ double tmp[NP];
    block_reduce_to_slot<NP>(v, tmp);
    __syncthreads();
    #pragma unroll
    for (int k = 0; k < NP; ++k) out[k] = tmp[k];
}

__device__ __forceinline__ void set_cond(cudaGraphConditionalHandle h, bool more) {
    if (h) cudaGraphSetConditional(h, more ? 1u : 0u);
}

__device__ __forceinline__ bool iteration_done(Ctrl* c, double res) {
    c->residual = res;
    c->iter += 1;
    bool done;
    if (c->fixed_iters > 0) done = c->iter >= c->fixed_iters;
    else done = (res < c->tol) || (c->iter >= c->max_iter);
    c->done = done ? 1 : 0;
    return done;
}

// ------------------------------------------------------------------ PageRank / RWR epilogue
struct EpiAffine {
    float* y; float* p; float* z_next; const float* inv_deg;
    Ctrl* ctrl; double* slots; int32_t slot_base, total_slots, is_last;
    cudaGraphConditionalHandle cond;
    int32_t rwr;
    // per thread
    float c, tele; int32_t q; double res, dm;

    __device__ __forceinline__ bool begin() {
        if (*(volatile int32_t*)&ctrl->done) return false;
        c = (float)ctrl->c; tele = (float)ctrl->tele; q = ctrl->q;
        res = 0.0; dm = 0.0;
        return true;
    }
    __device__ __forceinline__ void write(uint32_t ent, float v) {
        const uint32_t r = ent & ROW_MASK;
        if (ent & FLAG_ACC) v += y[r];
        if (!(ent & FLAG_FINAL)) { y[r] = v; return; }
        float pn = fmaf(c, v, tele);
        if (rwr && (int32_t)r == q) pn += 1.0f - c;
        const float po = p[r];
        res += fabs((double)pn - (double)po);
        p[r] = pn;
        const float id = __ldg(inv_deg + r);
        z_next[r] = pn * id;
        if (id == 0.0f) dm += (double)pn;
    }
    __device__ __forceinline__ void end() {
        double v[2] = {res, dm};
        block_reduce_to_slot<2>(v, slots + 2 * (size_t)(slot_base + blockIdx.x));
        if (!is_last) return;
        if (!last_block(&ctrl->ticket)) return;
        double s[2];
        block_sum_slots<2>(slots, total_slots, s);
        if (threadIdx.x == 0) {
            ctrl->ticket = 0;
            // next iteration's additive term: PageRank c*D/n + (1-c)/n (reading R1); RWR 0
            if (!rwr) ctrl->tele = ctrl->c * s[1] * ctrl->inv_n + (1.0 - ctrl->c) * ctrl->inv_n;
            ctrl->dmass = s[1];
            bool done = iteration_done(ctrl, s[0]);
            __threadfence();
            set_cond(cond, !done);
        }
    }
};

// ------------------------------------------------------------------ HITS epilogues
struct EpiHitsSpmv {
    float* y; const uint8_t* half;
    Ctrl* ctrl; double* slots; int32_t slot_base, total_slots, is_last, l2;
    double s0, s1;
    __device__ __forceinline__ bool begin() {
        if (*(volatile int32_t*)&ctrl->done) return false;
        s0 = 0.0; s1 = 0.0;
        return true;
    }
    __device__ __forceinline__ void write(uint32_t ent, float v) {
        const uint32_t r = ent & ROW_MASK;
        if (ent & FLAG_ACC) v += y[r];
        y[r] = v;
        if (!(ent & FLAG_FINAL)) return;
        const double d = l2 ? (double)v * (double)v : fabs((double)v);
        if (__ldg(half + r)) s1 += d; else s0 += d;
    }
    __device__ __forceinline__ void end() {
        double v[2] = {s0, s1};
        block_reduce_to_slot<2>(v, slots + 2 * (size_t)(slot_base + blockIdx.x));
        if (!is_last) return;
        if (!last_block(&ctrl->ticket)) return;
        double s[2];
        block_sum_slots<2>(slots, total_slots, s);
        if (threadIdx.x == 0) {
            ctrl->ticket = 0;
            ctrl->norm[0] = l2 ? sqrt(s[0]) : s[0];
            ctrl->norm[1] = l2 ? sqrt(s[1]) : s[1];
        }
    }
};

// a' = y_a / |y_a|, h' = y_h / |y_h| (zero half -> uniform, reading R5); L1 change accumulated
__global__ void __launch_bounds__(kThreads) hits_normalize(const float* __restrict__ y,
                                                           float* __restrict__ v,
                                                           const uint8_t* __restrict__ half,
                                                           int64_t N, Ctrl* ctrl, double* slots,
                                                           cudaGraphConditionalHandle cond) {
    if (*(volatile int32_t*)&ctrl->done) return;
    const double n0 = ctrl->norm[0], n1 = ctrl->norm[1];
    const float uni = (float)ctrl->uniform;
    const float s0 = n0 > 0.0 ? (float)(1.0 / n0) : 0.0f, s1 = n1 > 0.0 ? (float)(1.0 / n1) : 0.0f;
    double res = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < N; i += (int64_t)gridDim.x * kThreads) {
        const int h = half[i];
        const double nn = h ? n1 : n0;
        const float vn = nn > 0.0 ? y[i] * (h ? s1 : s0) : uni;
        res += fabs((double)vn - (double)v[i]);
        v[i] = vn;
    }
    double acc[1] = {res};
    block_reduce_to_slot<1>(acc, slots + blockIdx.x);
    if (!last_block(&ctrl->ticket)) return;
    double s[1];
    block_sum_slots<1>(slots, gridDim.x, s);
    if (threadIdx.x == 0) {
        ctrl->ticket = 0;
        bool done = iteration_done(ctrl, s[0]);
        __threadfence();
        set_cond(cond, !done);
    }
}

__global__ void init_affine(float* p, float* z, const float* inv_deg, int64_t n, int32_t rwr,
                            int32_t q, float p0) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        float v = rwr ? (i == q ? 1.0f : 0.0f) : p0;
        p[i] = v;
        z[i] = v * inv_deg[i];
    }
}
__global__ void init_fill(float* v, int64_t n, float val) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        v[i] = val;
}

// ------------------------------------------------------------------ host: graph matrices
// counting sort permutation of [0,N) by (len desc, id asc): pi[id] = new position
static void order_by_length(const std::vector<int64_t>& len, std::vector<int32_t>& pi) {
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
static void clean_adjacency(int64_t n, const int64_t* rp, const int32_t* col,
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
static void relabel_csr(int64_t N, const std::vector<int64_t>& rp, const std::vector<int32_t>& col,
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
static void transpose(int64_t n, const std::vector<int64_t>& rp, const std::vector<int32_t>& col,
                      std::vector<int64_t>& trp, std::vector<int32_t>& tcol) {
    trp.assign(n + 1, 0);
    for (int64_t k = 0; k < rp[n]; ++k) trp[col[k] + 1]++;
    for (int64_t i = 0; i < n; ++i) trp[i + 1] += trp[i];
    tcol.resize(rp[n]);
    std::vector<int64_t> pos(trp.begin(), trp.end() - 1);
    for (int64_t u = 0; u < n; ++u)
        for (int64_t k = rp[u]; k < rp[u + 1]; ++k) tcol[pos[col[k]]++] = (int32_t)u;
}

}  // namespace tc

using namespace tc;

// ------------------------------------------------------------------ solver object
static spmv_status build_solver(spmv_solver_s* s, const int64_t* row_ptr, const int32_t* col,
                                const spmv_options* opt_in) {
    const int64_t n = s->n;
    std::vector<int64_t> arp; std::vector<int32_t> acol;
    clean_adjacency(n, row_ptr, col, arp, acol);
    std::vector<int64_t> len;           // column length of the iteration matrix (relabel key)
    std::vector<int64_t> mrp;           // iteration matrix in original ids
    std::vector<int32_t> mcol;
    std::vector<float> inv_deg;
    if (s->algo == SPMV_ALGO_PAGERANK) {
        transpose(n, arp, acol, mrp, mcol);                       // M = A^T
        len.resize(n);
        for (int64_t u = 0; u < n; ++u) len[u] = arp[u + 1] - arp[u];   // column u of A^T = outdeg
        s->N = n;
    } else if (s->algo == SPMV_ALGO_RWR) {
        std::vector<int64_t> trp; std::vector<int32_t> tcol;
        transpose(n, arp, acol, trp, tcol);
        mrp.assign(n + 1, 0);
        std::vector<std::vector<int32_t>> tmp;                    // S = binary(A u A^T)
        std::vector<int64_t> slen(n);
        mcol.clear();
        std::vector<int32_t> buf;
        mcol.reserve(2 * arp[n]);
        for (int64_t i = 0; i < n; ++i) {
            buf.assign(acol.begin() + arp[i], acol.begin() + arp[i + 1]);
            buf.insert(buf.end(), tcol.begin() + trp[i], tcol.begin() + trp[i + 1]);
            std::sort(buf.begin(), buf.end());
            buf.erase(std::unique(buf.begin(), buf.end()), buf.end());
            mcol.insert(mcol.end(), buf.begin(), buf.end());
            mrp[i + 1] = (int64_t)mcol.size();
        }
        len.resize(n);
        for (int64_t u = 0; u < n; ++u) len[u] = mrp[u + 1] - mrp[u];  // symmetric: col len = deg
        s->N = n;
    } else {
        // B = [[0, A^T], [A, 0]]: row v (< n) lists n+u for u->v; row n+u lists v for u->v
        std::vector<int64_t> trp; std::vector<int32_t> tcol;
        transpose(n, arp, acol, trp, tcol);
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
        for (int64_t k = 0; k < mrp[N]; ++k) len[mcol[k]]++;   // column lengths of B
        s->N = N;
    }
    const int64_t N = s->N;
    order_by_length(len, s->pi);
    Coo M;
    relabel_csr(N, mrp, mcol, s->pi, M);
    std::vector<float> invd_pi(N, 0.0f);
    std::vector<uint8_t> half_pi;
    int64_t n_dangling = 0;
    if (s->algo == SPMV_ALGO_HITS) {
        half_pi.assign(N, 0);
        for (int64_t i = n; i < N; ++i) half_pi[s->pi[i]] = 1;
    } else {
        for (int64_t u = 0; u < n; ++u) {
            invd_pi[s->pi[u]] = len[u] ? (float)(1.0 / (double)len[u]) : 0.0f;
            n_dangling += (len[u] == 0);
        }
    }
    s->n_dangling = n_dangling;
    spmv_options opt;
    if (opt_in) opt = *opt_in; else spmv_options_default(&opt);
    opt.pattern = 1;
    spmv_status st = create_plan(N, N, (int64_t)M.col.size(), M.rp.data(), M.col.data(), nullptr,
                                 &opt, s->device, &s->plan);
    if (st) return st;
    spmv_plan_s* p = s->plan;
    cudaError_t e;
#define CKE(x) do { if ((e = (x)) != cudaSuccess) return cuda_status(e, #x); } while (0)
    CKE(cudaMalloc(&s->d_p, N * sizeof(float)));
    CKE(cudaMalloc(&s->d_y, N * sizeof(float)));
    CKE(cudaMalloc(&s->d_z[0], N * sizeof(float)));
    CKE(cudaMalloc(&s->d_z[1], N * sizeof(float)));
    CKE(cudaMalloc(&s->d_inv, N * sizeof(float)));
    CKE(cudaMemcpy(s->d_inv, invd_pi.data(), N * sizeof(float), cudaMemcpyHostToDevice));
    CKE(cudaMalloc(&s->d_half, std::max<int64_t>(N, 1)));
    if (!half_pi.empty()) CKE(cudaMemcpy(s->d_half, half_pi.data(), N, cudaMemcpyHostToDevice));
    CKE(cudaMalloc(&s->d_ctrl, sizeof(Ctrl)));
    CKE(cudaMemset(s->d_ctrl, 0, sizeof(Ctrl)));
    // launches and partial slots
    if (s->algo == SPMV_ALGO_HITS) CKE(setup_grids<EpiHitsSpmv>(*p, s->grids));
    else CKE(setup_grids<EpiAffine>(*p, s->grids));
    s->tiles_used.clear();
    s->slot_base.clear();
    int32_t slots = 0;
    for (int32_t t = 0; t <= p->num_tiles; ++t) {
        if (p->tiles[t].wl_end == p->tiles[t].wl_begin) continue;
        s->tiles_used.push_back(t);
        s->slot_base.push_back(slots);
        slots += s->grids[t];
    }
    s->total_slots = slots;
    s->norm_grid = p->sm_count * 4;
    CKE(cudaMalloc(&s->d_slots, (size_t)std::max(slots, s->norm_grid) * 2 * sizeof(double)));
#undef CKE
    return SPMV_OK;
}

// enqueue one iteration reading z_in (PR/RWR) and writing z_out
static cudaError_t enqueue_iteration(spmv_solver_s* s, int parity, cudaStream_t st,
                                     cudaGraphConditionalHandle cond) {
    spmv_plan_s* p = s->plan;
    const size_t nu = s->tiles_used.size();
    if (s->algo == SPMV_ALGO_HITS) {
        for (size_t i = 0; i < nu; ++i) {
            EpiHitsSpmv epi{};
            epi.y = s->d_y; epi.half = s->d_half; epi.ctrl = s->d_ctrl; epi.slots = s->d_slots;
            epi.slot_base = s->slot_base[i]; epi.total_slots = s->total_slots;
            epi.is_last = (i + 1 == nu); epi.l2 = s->it.hits_norm != 1;
            cudaError_t e = launch_tile(*p, s->tiles_used[i], s->grids[s->tiles_used[i]], s->d_p, epi, st);
            if (e) return e;
        }
        hits_normalize<<<s->norm_grid, kThreads, 0, st>>>(s->d_y, s->d_p, s->d_half, s->N, s->d_ctrl,
                                                           s->d_slots, cond);
        return cudaGetLastError();
    }
    for (size_t i = 0; i < nu; ++i) {
        EpiAffine epi{};
        epi.y = s->d_y; epi.p = s->d_p; epi.z_next = s->d_z[parity ^ 1]; epi.inv_deg = s->d_inv;
        epi.ctrl = s->d_ctrl; epi.slots = s->d_slots; epi.slot_base = s->slot_base[i];
        epi.total_slots = s->total_slots; epi.is_last = (i + 1 == nu); epi.cond = cond;
        epi.rwr = s->algo == SPMV_ALGO_RWR;
        cudaError_t e = launch_tile(*p, s->tiles_used[i], s->grids[s->tiles_used[i]], s->d_z[parity], epi, st);
        if (e) return e;
    }
    return cudaSuccess;
}

static spmv_status build_graph(spmv_solver_s* s, cudaStream_t st) {
    cudaError_t e;
    cudaGraph_t g = nullptr;
    if ((e = cudaGraphCreate(&g, 0))) return cuda_status(e, "cudaGraphCreate");
    cudaGraphConditionalHandle h;
    if ((e = cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault)))
        return cuda_status(e, "cudaGraphConditionalHandleCreate");
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    if ((e = cudaGraphAddNode(&node, g, nullptr, 0, &cp))) return cuda_status(e, "cudaGraphAddNode");
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    if ((e = cudaStreamBeginCaptureToGraph(st, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed)))
        return cuda_status(e, "cudaStreamBeginCaptureToGraph");
    cudaError_t e1 = enqueue_iteration(s, 0, st, h);
    cudaError_t e2 = (s->algo == SPMV_ALGO_HITS) ? cudaSuccess : enqueue_iteration(s, 1, st, h);
    cudaGraph_t captured = nullptr;
    e = cudaStreamEndCapture(st, &captured);
    if (e1) return cuda_status(e1, "capture iteration");
    if (e2) return cuda_status(e2, "capture iteration");
    if (e) return cuda_status(e, "cudaStreamEndCapture");
    if ((e = cudaGraphInstantiate(&s->exec, g, 0))) return cuda_status(e, "cudaGraphInstantiate");
    s->graph = g;
    return SPMV_OK;
}

extern "C" {

__attribute__((visibility("default"))) void spmv_iter_opts_default(spmv_iter_opts* o, int algo) {
    if (!o) return;
    o->c = algo == SPMV_ALGO_RWR ? 0.9 : 0.85;
    o->tol = 1e-6; o->max_iter = 1000; o->hits_norm = 2; o->fixed_iters = 0;
}

__attribute__((visibility("default")))
spmv_status spmv_solver_create(int algo, int64_t n, int64_t m, const int64_t* row_ptr,
                               const int32_t* col, const spmv_iter_opts* it,
                               const spmv_options* opt, spmv_comm comm, int device,
                               spmv_solver* out) {
    if (!out || !row_ptr || (m > 0 && !col) || n < 1) { set_error("invalid argument"); return SPMV_EINVAL; }
    if (algo < 0 || algo > 2) { set_error("unknown algorithm"); return SPMV_EINVAL; }
    if (row_ptr[0] != 0 || row_ptr[n] != m) { set_error("row_ptr inconsistent with m"); return SPMV_EINVAL; }
    for (int64_t i = 0; i < n; ++i) if (row_ptr[i + 1] < row_ptr[i]) { set_error("row_ptr not monotone"); return SPMV_EINVAL; }
    for (int64_t k = 0; k < m; ++k) if (col[k] < 0 || col[k] >= n) { set_error("target out of range"); return SPMV_EINVAL; }
    if (algo == SPMV_ALGO_HITS && 2 * n >= (int64_t(1) << 29)) { set_error("2n must be < 2^29"); return SPMV_ERANGE; }
    if (device < 0) { set_error("solvers need a device"); return SPMV_EINVAL; }
    if (comm) return solver_create_dist(algo, n, m, row_ptr, col, it, opt, comm, device, out);
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) { set_error("no CUDA device"); return SPMV_ECUDA; }
    cudaError_t e = cudaSetDevice(device);
    if (e) return cuda_status(e, "cudaSetDevice");
    spmv_solver_s* s = new spmv_solver_s();
    s->algo = algo; s->n = n; s->device = device;
    if (it) s->it = *it; else spmv_iter_opts_default(&s->it, algo);
    spmv_status st;
    try {
        st = build_solver(s, row_ptr, col, opt);
    } catch (const std::bad_alloc&) {
        st = SPMV_ENOMEM; set_error("host allocation failed");
    }
    if (st) { spmv_solver_destroy(s); return st; }
    *out = s;
    return SPMV_OK;
}

__attribute__((visibility("default")))
spmv_status spmv_solver_run(spmv_solver s, int64_t query, void* stream, spmv_iter_result* res) {
    if (!s) { set_error("null solver"); return SPMV_EINVAL; }
    if (s->comm) return solver_run_dist(s, query, stream, res);
    if (s->algo == SPMV_ALGO_RWR && (query < 0 || query >= s->n)) { set_error("query out of range"); return SPMV_ERANGE; }
    cudaError_t e = cudaSetDevice(s->device);
    if (e) return cuda_status(e, "cudaSetDevice");
    cudaStream_t st = (cudaStream_t)stream;
    if (!st) {
        if (!s->own_stream && (e = cudaStreamCreateWithFlags(&s->own_stream, cudaStreamNonBlocking)))
            return cuda_status(e, "stream");
        st = s->own_stream;
    }
    if (!s->exec) { spmv_status b = build_graph(s, st); if (b) return b; }
    Ctrl c{};
    const double n = (double)s->n;
    c.c = s->it.c; c.tol = s->it.tol; c.max_iter = s->it.max_iter; c.fixed_iters = s->it.fixed_iters;
    c.inv_n = 1.0 / n; c.iter = 0; c.done = 0; c.ticket = 0; c.residual = INFINITY;
    c.q = (s->algo == SPMV_ALGO_RWR) ? s->pi[query] : -1;
    c.uniform = s->it.hits_norm == 1 ? 1.0 / n : 1.0 / std::sqrt(n);
    if (s->algo == SPMV_ALGO_PAGERANK) {
        double D0 = (double)s->n_dangling / n;                 // p(0) = 1/n
        c.tele = c.c * D0 / n + (1.0 - c.c) / n;
    } else c.tele = 0.0;
    if ((e = cudaMemcpyAsync(s->d_ctrl, &c, sizeof(Ctrl), cudaMemcpyHostToDevice, st))) return cuda_status(e, "ctrl");
    const int g = s->plan->sm_count * 4;
    if (s->algo == SPMV_ALGO_HITS) init_fill<<<g, 256, 0, st>>>(s->d_p, s->N, (float)(1.0 / n));
    else init_affine<<<g, 256, 0, st>>>(s->d_p, s->d_z[0], s->d_inv, s->N, s->algo == SPMV_ALGO_RWR,
                                         (int32_t)c.q, (float)(1.0 / n));
    if ((e = cudaGetLastError())) return cuda_status(e, "init");
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0, st);
    e = cudaGraphLaunch(s->exec, st);
    cudaEventRecord(e1, st);
    if (e) { cudaEventDestroy(e0); cudaEventDestroy(e1); return cuda_status(e, "cudaGraphLaunch"); }
    if ((e = cudaMemcpyAsync(&c, s->d_ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, st)) ||
        (e = cudaStreamSynchronize(st))) {
        cudaEventDestroy(e0); cudaEventDestroy(e1); return cuda_status(e, "iteration loop");
    }
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0); cudaEventDestroy(e1);
    s->last = c;
    if (res) {
        res->iterations = c.iter; res->residual = c.residual;
        res->converged = s->it.fixed_iters > 0 ? 1 : (c.residual < s->it.tol);
        res->ms_total = ms; res->us_per_iter = c.iter ? 1000.0 * ms / c.iter : 0.0;
        res->predicted_us_per_iter = s->plan->predicted_us;
    }
    if (s->it.fixed_iters <= 0 && !(c.residual < s->it.tol)) { set_error("max_iter reached"); return SPMV_ENOCONV; }
    return SPMV_OK;
}

__attribute__((visibility("default")))
spmv_status spmv_solver_result(spmv_solver s, float* out0, float* out1) {
    if (!s || !out0 || (s->algo == SPMV_ALGO_HITS && !out1)) { set_error("null argument"); return SPMV_EINVAL; }
    if (s->comm) return solver_result_dist(s, out0, out1);
    std::vector<float> v(s->N);
    cudaSetDevice(s->device);
    cudaError_t e = cudaMemcpy(v.data(), s->d_p, s->N * sizeof(float), cudaMemcpyDeviceToHost);
    if (e) return cuda_status(e, "result");
    for (int64_t u = 0; u < s->n; ++u) out0[u] = v[s->pi[u]];
    if (s->algo == SPMV_ALGO_HITS)
        for (int64_t u = 0; u < s->n; ++u) out1[u] = v[s->pi[s->n + u]];
    return SPMV_OK;
}

__attribute__((visibility("default")))
spmv_status spmv_solver_plan_stats(spmv_solver s, spmv_plan_stats_t* out) {
    if (!s || !s->plan) { set_error("null solver"); return SPMV_EINVAL; }
    return spmv_plan_stats(s->plan, out);
}

__attribute__((visibility("default"))) int32_t spmv_solver_launches_per_iter(spmv_solver s) {
    if (!s) return 0;
    return (int32_t)s->tiles_used.size() + (s->algo == SPMV_ALGO_HITS ? 1 : 0);
}

__attribute__((visibility("default"))) void spmv_solver_destroy(spmv_solver s) {
    if (!s) return;
    if (s->comm) { solver_destroy_dist(s); return; }
    cudaSetDevice(s->device);
    if (s->exec) cudaGraphExecDestroy(s->exec);
    if (s->graph) cudaGraphDestroy(s->graph);
    if (s->own_stream) cudaStreamDestroy(s->own_stream);
    cudaFree(s->d_p); cudaFree(s->d_y); cudaFree(s->d_z[0]); cudaFree(s->d_z[1]); cudaFree(s->d_inv);
    cudaFree(s->d_half); cudaFree(s->d_ctrl); cudaFree(s->d_slots);
    if (s->plan) spmv_plan_destroy(s->plan);
    delete s;
}

static spmv_status one_shot(int algo, int64_t n, int64_t m, const int64_t* rp, const int32_t* col,
                            int64_t query, const spmv_iter_opts* it, const spmv_options* opt,
                            spmv_comm comm, int device, float* o0, float* o1, spmv_iter_result* res) {
    spmv_solver s = nullptr;
    spmv_status st = spmv_solver_create(algo, n, m, rp, col, it, opt, comm, device, &s);
    if (st) return st;
    spmv_status r = spmv_solver_run(s, query, nullptr, res);
    if (r == SPMV_OK || r == SPMV_ENOCONV) {
        spmv_status q = spmv_solver_result(s, o0, o1);
        if (q) r = q;
    }
    spmv_solver_destroy(s);
    return r;
}

__attribute__((visibility("default")))
spmv_status pagerank(int64_t n, int64_t m, const int64_t* rp, const int32_t* col,
                     const spmv_iter_opts* it, const spmv_options* opt, spmv_comm comm, int device,
                     float* p_out, spmv_iter_result* res) {
    return one_shot(SPMV_ALGO_PAGERANK, n, m, rp, col, 0, it, opt, comm, device, p_out, nullptr, res);
}
__attribute__((visibility("default")))
spmv_status hits(int64_t n, int64_t m, const int64_t* rp, const int32_t* col,
                 const spmv_iter_opts* it, const spmv_options* opt, spmv_comm comm, int device,
                 float* a_out, float* h_out, spmv_iter_result* res) {
    return one_shot(SPMV_ALGO_HITS, n, m, rp, col, 0, it, opt, comm, device, a_out, h_out, res);
}
__attribute__((visibility("default")))
spmv_status rwr(int64_t n, int64_t m, const int64_t* rp, const int32_t* col, int64_t query,
                const spmv_iter_opts* it, const spmv_options* opt, spmv_comm comm, int device,
                float* r_out, spmv_iter_result* res) {
    return one_shot(SPMV_ALGO_RWR, n, m, rp, col, query, it, opt, comm, device, r_out, nullptr, res);
}

}  // extern "C"
