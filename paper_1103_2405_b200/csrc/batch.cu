// batch.cu -- batched Random Walk with Restart (the
// paper averages 25 random query nodes).  The Q <= 32 queries iterate together as one SpMM
// Y = W R over a row-major-only (CSR-vector, f2) tiled-composite layout of the same matrix: lanes
// are queries, so every stored entry costs one coalesced 128-byte read of an x row (all queries'
// values of that column) instead of a random 4-byte gather per query.  A warp walks a workload's
// slots as one flat stream with 16 x-row loads in flight whatever the row lengths, and writes
// each finished row of Y (stores only); Eq. 9 runs as a separate streaming pass over the N x 32
// rows (spmm_rwr_epilogue: r' = c y + (1-c) e_q, z' = r' / deg, per-query fp64 L1 change reduced
// in a fixed order), then the device-side WHILE loop decides.  Split rows combine in chunk order.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "epilogues.cuh"
#include "graph_build.h"
#include "launch.cuh"
#include "solver.h"

namespace tc {

constexpr int kQP = 32;                 // padded queries per row (one per lane)
constexpr int kBatchCtasPerSm = 2;      // spmm_rwr_tile: 2 x 512 threads per SM (<= 64 registers)

struct BatchArgs {
    const WlDesc* desc;
    int64_t wl_begin, wl_end;
    const int32_t* col;
    const uint32_t* row_id;
    int64_t col_lo;                     // tile's first relabelled column
    int32_t width;                      // sentinel
    const int32_t* split;               // [n_split][3]
    float* partials;                    // [n_chunks][32]
    int32_t* counters;                  // [n_split]
    const float* Z;                     // [N][32] input (r * inv_deg)
    float* Znext;                       // [N][32]
    float* R;                           // [N][32] current iterate (updated in place)
    float* Y;                           // [N][32] partial sums of rows shared by several tiles
    const float* inv;                   // [N]
    const int32_t* q;                   // [32] relabelled query per lane (-1: padding lane)
    float c;
    Ctrl* ctrl;
    double* slots;                      // [grid][32] per-block residual partials
    double* res_out;                    // [32]
    int32_t slot_base, total_slots, is_last;
    cudaGraphConditionalHandle cond;
    int64_t zero_row;                   // a row of Z that is always zero (row N: padding, never written)
};

// The SpMM writes the product Y = W_pattern Z only (first touch stores, later tiles add): its
// stores need no response, so a warp's gathers never wait on epilogue traffic.  Eq. 9 is applied
// by spmm_rwr_epilogue, a streaming pass over the N x 32 rows.
struct BatchEpi {
    const BatchArgs& a;
    int lane;
    __device__ __forceinline__ void write(uint32_t ent, float v) {
        if (ent == PAD_ROW) return;
        const int64_t o = (int64_t)(ent & ROW_MASK) * kQP + lane;
        if (ent & FLAG_ACC) v += a.Y[o];
        a.Y[o] = v;
    }
};

// the x row of tile column c; the padding sentinel reads the zero row, so the load is
// unconditional (a select on the loaded value made the compiler retire each load before issuing
// the next one into the same register: profiles/r02_batch_rwr_tuning.log, run97)
__device__ __forceinline__ float xrow(const BatchArgs& a, int32_t c, int lane) {
    const int64_t row = c != a.width ? a.col_lo + c : a.zero_row;
    return __ldg(a.Z + row * kQP + lane);
}

#ifndef TC_BATCH_U
#define TC_BATCH_U 16
#endif
constexpr int kRowU = TC_BATCH_U;       // x-row loads in flight per warp step
static_assert(32 % kRowU == 0, "a step must not straddle the 32 column ids a warp holds");

// row rr of a column-major 32-row slab (k-interleaved by kvec): its w slots sit at
// sb + (k / kvec) * 32 kvec + rr kvec + k % kvec; 32 ids per warp load, then as row_dot
__device__ __forceinline__ float slab_row_dot(const BatchArgs& a, const int32_t* sb, int rr, int w, int kvec,
                                              int lane) {
    float acc = 0.0f;
    for (int k0 = 0; k0 < w; k0 += 32) {
        const int k = k0 + lane;
        const int32_t cl = k < w ? __ldg(sb + (k / kvec) * 32 * kvec + rr * kvec + k % kvec) : a.width;
        const int n = min(32, w - k0);
        for (int j0 = 0; j0 < n; j0 += kRowU) {
            float xv[kRowU];
            #pragma unroll
            for (int t = 0; t < kRowU; ++t) xv[t] = xrow(a, __shfl_sync(0xffffffffu, cl, j0 + t), lane);
            #pragma unroll
            for (int t = 0; t < kRowU; ++t) acc += xv[t];
        }
    }
    return acc;
}

// a split chunk's partial; the last chunk to arrive sums the row's chunks in chunk order
__device__ __forceinline__ void split_write(const BatchArgs& a, const WlDesc& d, uint32_t ent, float v,
                                            BatchEpi& epi, int lane) {
    const int32_t* sp = a.split + 3 * d.split_id;
    const int32_t nch = __ldg(sp + 1), pbase = __ldg(sp + 2);
    a.partials[(int64_t)(pbase + d.chunk) * kQP + lane] = v;
    __threadfence();
    __syncwarp();
    int32_t t = 0;
    if (lane == 0) t = atomicAdd(a.counters + d.split_id, 1);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t == nch - 1) {
        __threadfence();
        float s = 0.0f;
        for (int32_t c = 0; c < nch; ++c) s += __ldcg(a.partials + (int64_t)(pbase + c) * kQP + lane);
        __syncwarp();
        if (lane == 0) a.counters[d.split_id] = 0;
        epi.write(ent, s);
    }
}

__global__ void __launch_bounds__(512, 2) spmm_rwr_tile(BatchArgs a) {
    if (*(volatile int32_t*)&a.ctrl->done) return;
    const int lane = threadIdx.x & 31, warps = blockDim.x >> 5;
    const int64_t gw = (int64_t)blockIdx.x * warps + (threadIdx.x >> 5);
    const int64_t G = (int64_t)gridDim.x * warps;
    BatchEpi epi{a, lane};
    // x rows with plain L2 caching (evict-last / evict-first hints on the hub / tail rows measured
    // slower on c2, 5.5-6.6 vs 4.3 ms per iteration)
    for (int64_t j = a.wl_begin + gw; j < a.wl_end; j += G) {
        const WlDesc d = load_desc(a.desc + j);
        const int32_t* wc = a.col + d.off;
        if (d.kind != KIND_CM) {
            // the workload's h rows of w slots as one flat stream: kRowU x-row loads in flight per
            // step whatever the row lengths; a row ends every w slots (warp-uniform)
            const int total = d.h * d.w;
            float acc = 0.0f;
            int32_t cl = (lane < total) ? __ldcs(wc + lane) : a.width;   // ids of slots [s0, s0 + 32)
            int32_t cn = a.width;
            int row = 0, next_end = d.w;                  // slot after the current row
            for (int s0 = 0; s0 < total; s0 += kRowU) {
                const int base = s0 & 31;
                // the next 32 ids are requested a step ahead of their use
                if (base == 0) cn = (s0 + 32 + lane < total) ? __ldcs(wc + s0 + 32 + lane) : a.width;
                float xv[kRowU];
                #pragma unroll
                for (int t = 0; t < kRowU; ++t) xv[t] = xrow(a, __shfl_sync(0xffffffffu, cl, base + t), lane);
                if (next_end - s0 > kRowU) {              // no row ends in this step (warp-uniform)
                    #pragma unroll
                    for (int t = 0; t < kRowU; ++t) acc += xv[t];
                } else {
                    #pragma unroll
                    for (int t = 0; t < kRowU; ++t) {
                        if (s0 + t >= total) break;
                        acc += xv[t];
                        if (s0 + t + 1 == next_end) {
                            const uint32_t ent = __ldg(a.row_id + d.row_base + row);
                            if (d.kind == KIND_SPLIT) split_write(a, d, ent, acc, epi, lane);
                            else epi.write(ent, acc);
                            acc = 0.0f;
                            ++row;
                            next_end += d.w;
                        }
                    }
                }
                if (base + kRowU == 32) cl = cn;
            }
        } else {
            // column major (zero-length rows of the remainder; the batch plan is row major only)
            const int slabs = d.h >> 5;
            for (int sl = 0; sl < slabs; ++sl) {
                const int32_t* sb = wc + (int64_t)sl * 32 * d.w;
                const uint32_t myent = __ldg(a.row_id + d.row_base + sl * 32 + lane);
                for (int rr = 0; rr < 32; ++rr) {
                    const float v = slab_row_dot(a, sb, rr, d.w, d.kvec, lane);
                    epi.write(__shfl_sync(0xffffffffu, myent, rr), v);
                }
            }
        }
    }
}

// Eq. 9 over every (row, query): r' = c y + (1 - c) e_q, z' = r' / deg; per-query L1 change in
// fp64, reduced in a fixed order (per block over warps, then the last block over blocks).
__global__ void __launch_bounds__(512) spmm_rwr_epilogue(BatchArgs a, int64_t N) {
    if (*(volatile int32_t*)&a.ctrl->done) return;
    const int lane = threadIdx.x & 31, warps = blockDim.x >> 5;
    // thread = 4 queries (one float4) of a row; a warp covers 4 rows per step, 4 steps in flight
    const int g = lane & 7, sub = lane >> 3;
    int32_t q[4];
    #pragma unroll
    for (int k = 0; k < 4; ++k) q[k] = a.q[4 * g + k];
    double rk[4] = {0.0, 0.0, 0.0, 0.0};
    const int64_t wid = (int64_t)blockIdx.x * warps + (threadIdx.x >> 5), W = (int64_t)gridDim.x * warps;
    constexpr int kU = 4;
    for (int64_t r0 = 4 * wid * kU; r0 < N; r0 += 4 * W * kU) {
        float4 y[kU], rold[kU];
        float iv[kU];
        #pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int64_t r = r0 + 4 * u + sub;
            if (r < N) {
                y[u] = __ldcs(reinterpret_cast<const float4*>(a.Y + r * kQP) + g);
                rold[u] = *(reinterpret_cast<const float4*>(a.R + r * kQP) + g);
                iv[u] = __ldg(a.inv + r);
            }
        }
        #pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int64_t r = r0 + 4 * u + sub;
            if (r >= N) continue;
            float rn[4] = {a.c * y[u].x, a.c * y[u].y, a.c * y[u].z, a.c * y[u].w};
            const float ro[4] = {rold[u].x, rold[u].y, rold[u].z, rold[u].w};
            #pragma unroll
            for (int k = 0; k < 4; ++k) {
                if ((int32_t)r == q[k]) rn[k] += 1.0f - a.c;     // Eq. 9: + (1 - c) e_q
                rk[k] += fabs((double)rn[k] - (double)ro[k]);
            }
            *(reinterpret_cast<float4*>(a.R + r * kQP) + g) = make_float4(rn[0], rn[1], rn[2], rn[3]);
            *(reinterpret_cast<float4*>(a.Znext + r * kQP) + g) =
                make_float4(rn[0] * iv[u], rn[1] * iv[u], rn[2] * iv[u], rn[3] * iv[u]);
        }
    }
    // per query 4g + k: sum the four row lanes (sub) of the warp in a fixed order
    double res = 0.0;
    #pragma unroll
    for (int k = 0; k < 4; ++k) {
        double v = rk[k];
        v += __shfl_xor_sync(0xffffffffu, v, 8);
        v += __shfl_xor_sync(0xffffffffu, v, 16);
        rk[k] = v;
    }
    // lane l now reports query l = 4 g + k with g = l >> 2, k = l & 3 (held by lanes g, g + 8, ...)
    {
        const int gq = lane >> 2, kq = lane & 3;
        double mine = 0.0;
        #pragma unroll
        for (int k = 0; k < 4; ++k) {
            const double v = __shfl_sync(0xffffffffu, rk[k], gq);
            if (k == kq) mine = v;
        }
        res = mine;
    }
    __shared__ double red[16][32];
    const int w = threadIdx.x >> 5;
    red[w][lane] = res;
    __syncthreads();
    if (threadIdx.x < 32) {
        double t = 0.0;
        for (int k = 0; k < warps; ++k) t += red[k][threadIdx.x];
        a.slots[(int64_t)blockIdx.x * 32 + threadIdx.x] = t;
    }
    if (!last_block(&a.ctrl->ticket)) return;
    if (threadIdx.x < 32) {
        double t = 0.0;
        for (int b = 0; b < (int)gridDim.x; ++b) t += __ldcg(a.slots + (int64_t)b * 32 + threadIdx.x);
        a.res_out[threadIdx.x] = t;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        a.ctrl->ticket = 0;
        double worst = 0.0;
        for (int l = 0; l < 32; ++l)
            if (a.q[l] >= 0) worst = fmax(worst, a.res_out[l]);
        const bool done = iteration_done(a.ctrl, worst);
        __threadfence();
        set_cond(a.cond, !done);
    }
}

__global__ void spmm_init(float* R, float* Z, const float* inv, const int32_t* q, int64_t N) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N * kQP; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / kQP;
        const int l = (int)(i % kQP);
        const float v = (q[l] >= 0 && r == q[l]) ? 1.0f : 0.0f;   // r(0) = e_q (reading R7)
        R[i] = v;
        Z[i] = v * inv[r];
    }
}

}  // namespace tc

using namespace tc;

struct BatchState {
    spmv_plan_s* plan = nullptr;        // the batch's own tiling of the iteration matrix
    std::vector<int32_t> tiles;         // non-empty tiles of `plan`
    float *R = nullptr, *Z[2] = {nullptr, nullptr}, *Y = nullptr, *partials = nullptr;
    int32_t* q = nullptr;
    double *slots = nullptr, *res = nullptr;
    int32_t Q = 0;
    int64_t N = 0;
    std::vector<int> grids;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    std::vector<double> residual;
    // the batch's vertex space: the solver's, or (two-phase solver plans, whose graph keeps its
    // given order) relabelled by column length so the batch's one-pass tiles need no x permute
    std::vector<int32_t> pi;            // original vertex -> batch row
    float* inv = nullptr;               // 1/deg in batch order
    bool own_inv = false;
};

static BatchArgs batch_args(spmv_solver_s* s, BatchState* B, int32_t t, int parity, int32_t slot_base,
                            int32_t total_slots, bool is_last, cudaGraphConditionalHandle cond) {
    spmv_plan_s* p = B->plan;
    const TileInfo& ti = p->tiles[t];
    BatchArgs a{};
    a.desc = p->d_desc; a.wl_begin = ti.wl_begin; a.wl_end = ti.wl_end;
    a.col = p->d_col; a.row_id = p->d_row_id; a.col_lo = ti.col_lo;
    a.width = (int32_t)(ti.col_hi - ti.col_lo);
    a.split = p->d_split; a.partials = B->partials; a.counters = p->d_counters;
    a.Z = B->Z[parity]; a.Znext = B->Z[parity ^ 1]; a.R = B->R; a.Y = B->Y; a.inv = B->inv;
    a.q = B->q; a.c = (float)s->it.c; a.ctrl = s->d_ctrl; a.slots = B->slots; a.res_out = B->res;
    a.zero_row = B->N;                  // Z rows N .. N+3: zeroed at allocation, never written
    a.slot_base = slot_base; a.total_slots = total_slots; a.is_last = is_last; a.cond = cond;
    return a;
}

// The batch's plan: one tile (x rows are 128 bytes here; a dense tile would make every row it
// shares with the remainder a 128-byte read-modify-write, measured slower on c2), row major only.
// Built from the solver plan's layout (identical matrix; the column order is the same length
// order, so the plan permutation stays the identity).
static spmv_status build_batch_plan(spmv_solver_s* s, BatchState* B) {
    spmv_plan_s* p = s->plan;
    int64_t tw = 0;
    int32_t T = 0;
    {
        int l2 = 0;
        cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, s->device);
        tw = std::max<int64_t>(4096, (int64_t)(0.4 * l2) / (kQP * 4)) / 4096 * 4096;
        if (const char* e = std::getenv("TCSPMV_BATCH_TW")) tw = std::atoll(e);
        T = 0;   // one tile: a dense tile's partial rows cost a 128-byte read-modify-write each
                 // (measured on c2: 1 tile 4.26 ms, 2 tiles 5.19 ms, 3 tiles 6.06 ms per iteration)
        if (const char* e = std::getenv("TCSPMV_BATCH_TILES")) T = std::atoi(e);
        T = (int32_t)std::min<int64_t>(T, (p->n_cols + tw - 1) / std::max<int64_t>(tw, 1));
    }
    std::vector<int32_t> rows(std::max<int64_t>(p->nnz, 1)), cols(std::max<int64_t>(p->nnz, 1));
    spmv_status st = spmv_plan_to_coo(p, rows.data(), cols.data(), nullptr);
    if (st) return st;
    std::vector<int64_t> rp(p->n_rows + 1, 0);
    for (int64_t k = 0; k < p->nnz; ++k) rp[rows[k] + 1]++;
    for (int64_t i = 0; i < p->n_rows; ++i) rp[i + 1] += rp[i];
    std::vector<int32_t> col(std::max<int64_t>(p->nnz, 1));
    {
        std::vector<int64_t> fill(rp.begin(), rp.end() - 1);
        for (int64_t k = 0; k < p->nnz; ++k) col[fill[rows[k]]++] = cols[k];
    }
    rows = {}; cols = {};
    B->pi = s->pi;
    B->inv = s->d_inv;
    if (p->two_phase) {
        // symmetric relabel by column length (Solution 2, L66), composed with the solver's order
        std::vector<int64_t> clen(p->n_cols, 0);
        for (int64_t k = 0; k < p->nnz; ++k) clen[col[k]]++;
        std::vector<int32_t> sigma;
        order_by_length(clen, sigma);
        Coo R;
        relabel_csr(p->n_rows, rp, col, sigma, R);
        rp = std::move(R.rp); col = std::move(R.col);
        for (auto& v : B->pi) v = sigma[v];
        std::vector<float> inv(p->n_rows), inv_b(p->n_rows);
        cudaError_t e = cudaMemcpy(inv.data(), s->d_inv, p->n_rows * sizeof(float), cudaMemcpyDeviceToHost);
        if (e) return cuda_status(e, "batch inv");
        for (int64_t i = 0; i < p->n_rows; ++i) inv_b[sigma[i]] = inv[i];
        if ((e = cudaMalloc(&B->inv, std::max<int64_t>(p->n_rows, 1) * sizeof(float)))) { B->inv = nullptr; return cuda_status(e, "batch inv"); }
        B->own_inv = true;
        if ((e = cudaMemcpy(B->inv, inv_b.data(), p->n_rows * sizeof(float), cudaMemcpyHostToDevice))) return cuda_status(e, "batch inv");
    }
    spmv_options opt = p->opt;
    opt.pattern = 1; opt.workload_sizes = nullptr; opt.perf_table_path = nullptr;
    opt.tile_width = (int32_t)std::min<int64_t>(tw, INT32_MAX);
    opt.num_tiles = T;
    opt.stage_x = 0;
    opt.two_phase = 0;         // the SpMM kernel runs on the one-pass tile layout
    // row major workloads only (the CSR-vector case of the format, f2): a warp walks whole rows,
    // each slot one 128-byte x row for all queries; rows padded to 4 slots
    opt.orient = 1;
    opt.align_rm = 4;
    if (opt.workload_size <= 0) opt.workload_size = p->opt.workload_size > 0 ? p->opt.workload_size : 1024;
    st = create_plan(p->n_rows, p->n_cols, p->nnz, rp.data(), col.data(), nullptr, &opt, s->device, &B->plan);
    if (st) return st;
    for (int64_t k = 0; k < p->n_cols; ++k)
        if (B->plan->perm[k] != (int32_t)k) { set_error("internal: batch plan permutation"); return SPMV_EINVAL; }
    for (int32_t t = 0; t <= B->plan->num_tiles; ++t)
        if (B->plan->tiles[t].wl_end > B->plan->tiles[t].wl_begin) B->tiles.push_back(t);

    // the solver plan's host layout copy was only needed for the decode
    p->L.desc = {}; p->L.row_id = {}; p->L.slot_col = {}; p->L.slot_val = {}; p->L.split = {};
    p->host_valid = false;
    return SPMV_OK;
}

static cudaError_t enqueue_batch_iteration(spmv_solver_s* s, BatchState* B, int parity, cudaStream_t st,
                                           cudaGraphConditionalHandle cond) {
    const size_t nu = B->tiles.size();
    const int sms = B->plan->sm_count * kBatchCtasPerSm;
    int32_t total = 0;
    for (size_t i = 0; i < nu; ++i) total += sms;
    int32_t base = 0;
    for (size_t i = 0; i < nu; ++i) {
        BatchArgs a = batch_args(s, B, B->tiles[i], parity, base, total, i + 1 == nu, cond);
        spmm_rwr_tile<<<sms, 512, 0, st>>>(a);
        base += sms;
        cudaError_t e = cudaGetLastError();
        if (e) return e;
    }
    BatchArgs a = batch_args(s, B, B->tiles.empty() ? 0 : B->tiles.back(), parity, 0, 0, true, cond);
    spmm_rwr_epilogue<<<B->plan->sm_count * 4, 512, 0, st>>>(a, B->N);
    return cudaGetLastError();
}

extern "C" {

__attribute__((visibility("default")))
spmv_status spmv_solver_run_batch(spmv_solver s, const int64_t* queries, int32_t Q, void* stream,
                                  spmv_iter_result* res) {
    if (!s || !queries || Q < 1 || Q > kQP) { set_error("invalid argument (1 <= Q <= 32)"); return SPMV_EINVAL; }
    if (s->algo != SPMV_ALGO_RWR || s->comm) { set_error("batched runs are single-GPU RWR"); return SPMV_EINVAL; }
    for (int32_t i = 0; i < Q; ++i)
        if (queries[i] < 0 || queries[i] >= s->n) { set_error("query out of range"); return SPMV_ERANGE; }
    cudaError_t e = cudaSetDevice(s->device);
    if (e) return cuda_status(e, "cudaSetDevice");
    cudaStream_t st = (cudaStream_t)stream;
    if (!st) {
        if (!s->own_stream && (e = cudaStreamCreateWithFlags(&s->own_stream, cudaStreamNonBlocking)))
            return cuda_status(e, "stream");
        st = s->own_stream;
    }
    BatchState* B = static_cast<BatchState*>(s->batch);
    if (!B) {
        B = new BatchState();
        s->batch = B;
        B->N = s->N;
        spmv_status bs = build_batch_plan(s, B);
        if (!bs && B->tiles.empty()) { set_error("internal: batch plan has no tiles"); bs = SPMV_EINVAL; }
        // a failed build leaves nothing attached: the next call starts over
        if (bs) { batch_destroy(s); return bs; }
    }
    spmv_plan_s* p = B->plan;
    if (!B->R) {
        const size_t vec = (size_t)(s->N + 4) * kQP * sizeof(float);
        // any failure below releases the whole batch state (buffers, graph, plan)
#define CKB(x) do { if ((e = (x)) != cudaSuccess) { spmv_status r_ = cuda_status(e, #x); batch_destroy(s); return r_; } } while (0)
        CKB(cudaMalloc(&B->R, vec));
        CKB(cudaMalloc(&B->Z[0], vec));
        CKB(cudaMalloc(&B->Z[1], vec));
        CKB(cudaMemset(B->Z[0], 0, vec));
        CKB(cudaMemset(B->Z[1], 0, vec));
        CKB(cudaMalloc(&B->Y, vec));
        CKB(cudaMalloc(&B->partials, (size_t)std::max<int64_t>(p->n_chunks, 1) * kQP * sizeof(float)));
        CKB(cudaMalloc(&B->q, kQP * sizeof(int32_t)));
        const size_t nslots = (size_t)p->sm_count * 4;
        CKB(cudaMalloc(&B->slots, nslots * kQP * sizeof(double)));
        CKB(cudaMalloc(&B->res, kQP * sizeof(double)));
    }
    if (!B->exec && !s->it.host_loop) {
        // device-side loop: WHILE node around two iterations (double-buffered input)
        cudaGraph_t g;
        CKB(cudaGraphCreate(&g, 0));
        B->graph = g;
        cudaGraphConditionalHandle h;
        CKB(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = h;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        cudaGraphNode_t node;
        CKB(cudaGraphAddNode(&node, g, nullptr, 0, &cp));
        cudaGraph_t body = cp.conditional.phGraph_out[0];
        CKB(cudaStreamBeginCaptureToGraph(st, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
        cudaError_t e1 = enqueue_batch_iteration(s, B, 0, st, h);
        cudaError_t e2 = enqueue_batch_iteration(s, B, 1, st, h);
        cudaGraph_t cap = nullptr;
        e = cudaStreamEndCapture(st, &cap);
        if (!e) e = e1 ? e1 : e2;
        CKB(e);
        CKB(cudaGraphInstantiate(&B->exec, g, 0));
#undef CKB
    }
    B->Q = Q;
    std::vector<int32_t> hq(kQP, -1);
    for (int32_t i = 0; i < Q; ++i) hq[i] = B->pi[queries[i]];
    Ctrl c{};
    c.c = s->it.c; c.tol = s->it.tol; c.max_iter = s->it.max_iter; c.fixed_iters = s->it.fixed_iters;
    c.inv_n = 1.0 / (double)s->n; c.residual = INFINITY; c.q = -1;
    if ((e = cudaMemcpyAsync(B->q, hq.data(), kQP * sizeof(int32_t), cudaMemcpyHostToDevice, st)) ||
        (e = cudaMemcpyAsync(s->d_ctrl, &c, sizeof(Ctrl), cudaMemcpyHostToDevice, st)))
        return cuda_status(e, "upload");
    spmm_init<<<p->sm_count * 8, 256, 0, st>>>(B->R, B->Z[0], B->inv, B->q, s->N);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0, st);
    cudaEvent_t e_stop = nullptr;
    if (s->it.host_loop) {
        // host-enqueued iterations (profilers, sanitizers): batches of 8, then the stop flag
        const int cap = std::max(s->it.max_iter, s->it.fixed_iters) + 8;
        std::vector<cudaEvent_t> ev;
        int launched = 0;
        e = cudaSuccess;
        while (!e) {
            for (int b = 0; b < 8 && !e; ++b, ++launched) {
                e = enqueue_batch_iteration(s, B, launched & 1, st, 0);
                cudaEvent_t v;
                cudaEventCreate(&v);
                cudaEventRecord(v, st);
                ev.push_back(v);
            }
            if (!e) e = cudaMemcpyAsync(&c, s->d_ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, st);
            if (!e) e = cudaStreamSynchronize(st);
            if (e || c.done || launched > cap) break;
        }
        if (!e && !ev.empty()) {
            const int64_t last = std::min<int64_t>(std::max<int64_t>(c.iter - 1, 0), (int64_t)ev.size() - 1);
            e_stop = ev[last];
            ev[last] = nullptr;
        }
        for (auto v : ev) if (v) cudaEventDestroy(v);
    } else {
        e = cudaGraphLaunch(B->exec, st);
    }
    cudaEventRecord(e1, st);
    B->residual.assign(kQP, 0.0);
    if (!e) e = cudaMemcpyAsync(&c, s->d_ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, st);
    if (!e) e = cudaMemcpyAsync(B->residual.data(), B->res, kQP * sizeof(double), cudaMemcpyDeviceToHost, st);
    if (!e) e = cudaStreamSynchronize(st);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e_stop ? e_stop : e1);
    cudaEventDestroy(e0); cudaEventDestroy(e1);
    if (e_stop) cudaEventDestroy(e_stop);
    if (e) return cuda_status(e, "batched loop");
    if (res) {
        res->iterations = c.iter; res->residual = c.residual;
        res->converged = s->it.fixed_iters > 0 ? 1 : (c.residual < s->it.tol);
        res->ms_total = ms; res->us_per_iter = c.iter ? 1000.0 * ms / c.iter : 0.0;
        res->phase_us[0] = res->us_per_iter; res->phase_us[1] = res->phase_us[2] = 0.0;
        res->predicted_us_per_iter = p->predicted_us;
    }
    if (s->it.fixed_iters <= 0 && !(c.residual < s->it.tol)) { set_error("max_iter reached"); return SPMV_ENOCONV; }
    return SPMV_OK;
}

__attribute__((visibility("default")))
spmv_status spmv_solver_result_batch(spmv_solver s, float* out) {
    if (!s || !out || !s->batch) { set_error("no batched run"); return SPMV_EINVAL; }
    BatchState* B = static_cast<BatchState*>(s->batch);
    std::vector<float> R((size_t)s->N * kQP);
    cudaSetDevice(s->device);
    cudaError_t e = cudaMemcpy(R.data(), B->R, R.size() * sizeof(float), cudaMemcpyDeviceToHost);
    if (e) return cuda_status(e, "result");
    for (int32_t qi = 0; qi < B->Q; ++qi)
        for (int64_t u = 0; u < s->n; ++u) out[(size_t)qi * s->n + u] = R[(size_t)B->pi[u] * kQP + qi];
    return SPMV_OK;
}

}  // extern "C"

void batch_destroy(spmv_solver s) {
    BatchState* B = static_cast<BatchState*>(s->batch);
    if (!B) return;
    if (B->exec) cudaGraphExecDestroy(B->exec);
    if (B->graph) cudaGraphDestroy(B->graph);
    cudaFree(B->R); cudaFree(B->Z[0]); cudaFree(B->Z[1]); cudaFree(B->Y); cudaFree(B->partials);
    cudaFree(B->q); cudaFree(B->slots); cudaFree(B->res);
    if (B->own_inv) cudaFree(B->inv);
    if (B->plan) spmv_plan_destroy(B->plan);
    delete B;
    s->batch = nullptr;
}
