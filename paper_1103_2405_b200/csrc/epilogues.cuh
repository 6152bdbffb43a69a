// epilogues.cuh -- fused power-iteration epilogues and deterministic reductions (SURVEY.md 8(a)
// a11-a14), shared by the single-GPU solvers (iterate.cu) and the row-partitioned ones (dist.cu).
#pragma once
#include <cuda_runtime.h>

#include "solver.h"
#include "tc_kernels.cuh"

namespace tc {

// ------------------------------------------------------------------ device helpers
template <int NP>
__device__ __forceinline__ void block_reduce_to_slot(double (&v)[NP], double* slot) {
    __shared__ double red[kWarps][NP];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __syncwarp();
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
    // p and inv are kept in row-entry order (index of the row's FINAL entry; fpos maps a row to
    // it for split rows), so their reads/writes are coalesced; z_next is in vertex order (x).
    float* y; float* p; float* z_next; const float* inv_deg; const int32_t* fpos;
    Ctrl* ctrl; double* slots; int32_t slot_base, total_slots, is_last;
    cudaGraphConditionalHandle cond;
    int32_t rwr;
    double* dist_out;   // row-partitioned mode: the last block writes {sum |dp|, dangling mass} here
    // per thread
    float c, tele; int32_t q; double res, dm;

    __device__ __forceinline__ bool begin() {
        if (*(volatile int32_t*)&ctrl->done) return false;
        c = (float)ctrl->c; tele = (float)ctrl->tele; q = ctrl->q;
        res = 0.0; dm = 0.0;
        return true;
    }
    struct Pre { float acc, p_old, inv; };
    static constexpr bool kEntryState = true;    // p, 1/deg in entry order: prefetch_rm
    __device__ __forceinline__ int32_t slot(uint32_t ent, int32_t e) const {
        return e >= 0 ? e : __ldg(fpos + (ent & ROW_MASK));
    }
    __device__ __forceinline__ Pre prefetch(uint32_t ent, int32_t e) const {
        Pre q{0.0f, 0.0f, 0.0f};
        if (ent == PAD_ROW) return q;
        const uint32_t r = ent & ROW_MASK;
        if (ent & FLAG_ACC) q.acc = y[r];
        if (ent & FLAG_FINAL) { const int32_t s = slot(ent, e); q.p_old = p[s]; q.inv = __ldg(inv_deg + s); }
        return q;
    }
    __device__ __forceinline__ Pre prefetch_entry(int32_t e) const {
        Pre q{0.0f, 0.0f, 0.0f};
        if (e >= 0) { q.p_old = p[e]; q.inv = __ldg(inv_deg + e); }
        return q;
    }
    __device__ __forceinline__ Pre prefetch_rm(uint32_t ent, int32_t e, int32_t has_acc) const {
        Pre q{0.0f, 0.0f, 0.0f};
        if (e >= 0) { q.p_old = p[e]; q.inv = __ldg(inv_deg + e); }   // entry order: no wait on ent
        // ent (whose load may still be in flight) is looked at only where it decides a load
        if ((has_acc || e == -1) && ent != PAD_ROW) {
            if (has_acc && (ent & FLAG_ACC)) q.acc = y[ent & ROW_MASK];
            if (e == -1 && (ent & FLAG_FINAL)) { const int32_t s = slot(ent, e); q.p_old = p[s]; q.inv = __ldg(inv_deg + s); }
        }
        return q;
    }
    __device__ __forceinline__ void write(uint32_t ent, int32_t e, float v) { commit(ent, e, v, prefetch(ent, e)); }
    // two-phase tiles: the rows' p and 1/deg (entry order) into L2 ahead of the rows
    __device__ __forceinline__ void prefetch_rows(int64_t e0, int32_t n, uint64_t pol) const {
        prefetch_l2_range(p + e0, 4LL * n, pol);
        prefetch_l2_range(inv_deg + e0, 4LL * n, pol);
    }
    __device__ __forceinline__ void commit(uint32_t ent, int32_t e, float v, const Pre& pre) {
        const uint32_t r = ent & ROW_MASK;
        v += pre.acc;
        if (!(ent & FLAG_FINAL)) { y[r] = v; return; }
        float pn = fmaf(c, v, tele);
        if (rwr && (int32_t)r == q) pn += 1.0f - c;
        res += fabs((double)pn - (double)pre.p_old);
        p[slot(ent, e)] = pn;
        // a vertex without out-edges is an empty column of the iteration matrix: its z is never
        // read (and, row-partitioned, has no place in the exchanged slot)
        if (pre.inv != 0.0f) z_next[r] = pn * pre.inv;
        else dm += (double)pn;
    }
    __device__ __forceinline__ void end() {
        double v[2] = {res, dm};
        block_reduce_to_slot<2>(v, slots + 2 * (size_t)(slot_base + blockIdx.x));
        if (!is_last) return;
        if (!last_block(&ctrl->ticket)) return;
        double s[2];
        block_sum_slots<2>(slots, total_slots, s);
        if (dist_out) {
            if (threadIdx.x == 0) { ctrl->ticket = 0; dist_out[0] = s[0]; dist_out[1] = s[1]; }
            return;
        }
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
    float* y; const uint8_t* half;     // half: in row-entry order (fpos for split rows)
    const int32_t* fpos;
    double* dist_out;                  // row-partitioned mode: last block writes the raw half sums
    Ctrl* ctrl; double* slots; int32_t slot_base, total_slots, is_last, l2;
    double s0, s1;
    __device__ __forceinline__ bool begin() {
        if (*(volatile int32_t*)&ctrl->done) return false;
        s0 = 0.0; s1 = 0.0;
        return true;
    }
    struct Pre { float acc; int half; };
    static constexpr bool kEntryState = true;    // half flag in entry order: prefetch_rm
    __device__ __forceinline__ Pre prefetch(uint32_t ent, int32_t e) const {
        Pre q{0.0f, 0};
        if (ent == PAD_ROW) return q;
        const uint32_t r = ent & ROW_MASK;
        if (ent & FLAG_ACC) q.acc = y[r];
        if (ent & FLAG_FINAL) q.half = __ldg(half + (e >= 0 ? e : __ldg(fpos + r)));
        return q;
    }
    __device__ __forceinline__ Pre prefetch_entry(int32_t e) const {
        Pre q{0.0f, 0};
        if (e >= 0) q.half = __ldg(half + e);
        return q;
    }
    __device__ __forceinline__ Pre prefetch_rm(uint32_t ent, int32_t e, int32_t has_acc) const {
        Pre q{0.0f, 0};
        if (e >= 0) q.half = __ldg(half + e);                           // entry order: no wait on ent
        if ((has_acc || e == -1) && ent != PAD_ROW) {
            if (has_acc && (ent & FLAG_ACC)) q.acc = y[ent & ROW_MASK];
            if (e == -1 && (ent & FLAG_FINAL)) q.half = __ldg(half + __ldg(fpos + (ent & ROW_MASK)));
        }
        return q;
    }
    __device__ __forceinline__ void write(uint32_t ent, int32_t e, float v) { commit(ent, e, v, prefetch(ent, e)); }
    __device__ __forceinline__ void prefetch_rows(int64_t e0, int32_t n, uint64_t pol) const {
        prefetch_l2_range(half + e0, n, pol);
    }
    __device__ __forceinline__ void commit(uint32_t ent, int32_t, float v, const Pre& pre) {
        const uint32_t r = ent & ROW_MASK;
        v += pre.acc;
        y[r] = v;
        if (!(ent & FLAG_FINAL)) return;
        const double d = l2 ? (double)v * (double)v : fabs((double)v);
        if (pre.half) s1 += d; else s0 += d;
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
            if (dist_out) { dist_out[0] = s[0]; dist_out[1] = s[1]; return; }
            ctrl->norm[0] = l2 ? sqrt(s[0]) : s[0];
            ctrl->norm[1] = l2 ? sqrt(s[1]) : s[1];
        }
    }
};

// a' = y_a / |y_a|, h' = y_h / |y_h| (zero half -> uniform, reading R5); L1 change accumulated
static __global__ void __launch_bounds__(kThreads) hits_normalize(const float* __restrict__ y,
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

static __global__ void init_affine(float* p, float* z, const float* inv_deg, int64_t n, int32_t rwr,
                            int32_t q, float p0) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        float v = rwr ? (i == q ? 1.0f : 0.0f) : p0;
        p[i] = v;
        z[i] = v * inv_deg[i];
    }
}
// entry-ordered p: p_e[k] = p(0) of the row of FINAL entry k (PageRank 1/n, RWR e_q)
static __global__ void init_entries(float* p_e, const uint32_t* row_id, int64_t n_entries, int32_t rwr,
                                    int32_t q, float p0) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n_entries; k += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t ent = row_id[k];
        float v = 0.0f;
        if (ent != PAD_ROW && (ent & FLAG_FINAL)) v = rwr ? ((int32_t)(ent & ROW_MASK) == q ? 1.0f : 0.0f) : p0;
        p_e[k] = v;
    }
}

static __global__ void init_fill(float* v, int64_t n, float val) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        v[i] = val;
}

}  // namespace tc
