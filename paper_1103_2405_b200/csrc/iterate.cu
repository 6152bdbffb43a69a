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

#include "epilogues.cuh"
#include "graph_build.h"
#include "launch.cuh"
#include "pb_launch.cuh"
#include "solver.h"
#include "trace.h"
#include "tune.h"

namespace tc {

spmv_status create_plan(int64_t n_rows, int64_t n_cols, int64_t nnz, const int64_t* row_ptr,
                        const int32_t* col, const float* val, const spmv_options* opt_in,
                        int device, spmv_plan_s** out);

}  // namespace tc

using namespace tc;

// ------------------------------------------------------------------ solver object
static spmv_status build_solver(spmv_solver_s* s, const int64_t* row_ptr, const int32_t* col,
                                const spmv_options* opt_in) {
    Range r_build("spmv_solver_create");
    const int64_t n = s->n;
    std::vector<int64_t> arp; std::vector<int32_t> acol;
    clean_adjacency(n, row_ptr, col, arp, acol);
    std::vector<int64_t> len;           // column length of the iteration matrix (relabel key)
    std::vector<int64_t> mrp;           // iteration matrix in original ids
    std::vector<int32_t> mcol;
    s->N = build_iteration_matrix(s->algo, n, arp, acol, mrp, mcol, len);
    const int64_t N = s->N;
    spmv_options opt;
    if (opt_in) opt = *opt_in; else spmv_options_default(&opt);
    opt.pattern = 1;
    spmv_status st = SPMV_OK;
    // The graph is relabelled symmetrically by column length (Solution 2, L66, rows and columns:
    // the SpMV output is then directly the next input) and iterated on the one-pass tiles, unless
    // two-phase tiles are asked for (two_phase = 1): those need no relabel (pb.h) and keep the
    // rows in their given order (degree-sorted rows multiply their work items).  Measured on c2
    // the two-phase iteration is slower than the one-pass one (PageRank 379 vs
    // 343 us: the fused epilogue's per-row operand loads sit on the reduce's critical path), so
    // the model's default here stays one-pass.
    if (opt.two_phase == 1) {
        s->pi.resize(N);
        for (int64_t i = 0; i < N; ++i) s->pi[i] = (int32_t)i;
        Coo M0;
        relabel_csr(N, mrp, mcol, s->pi, M0);
        st = create_plan(N, N, (int64_t)M0.col.size(), M0.rp.data(), M0.col.data(), nullptr, &opt, s->device, &s->plan);
        if (st) return st;
        if (!s->plan->two_phase) { spmv_plan_destroy(s->plan); s->plan = nullptr; }
    }
    if (!s->plan) {
        order_by_length(len, s->pi);
        Coo M;
        relabel_csr(N, mrp, mcol, s->pi, M);
        opt.two_phase = 0;
        st = create_plan(N, N, (int64_t)M.col.size(), M.rp.data(), M.col.data(), nullptr, &opt, s->device, &s->plan);
        if (st) return st;
    }
    // HITS: the normalisation pass (y, half flag, v read and written: 13 B per element) is a
    // separate launch the SpMV model does not cover
    if (s->algo == SPMV_ALGO_HITS) s->pred_extra_us = stream_pass_us(opt, 13.0 * (double)N);
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
    spmv_plan_s* p = s->plan;
    cudaError_t e;
#define CKE(x) do { if ((e = (x)) != cudaSuccess) return cuda_status(e, #x); } while (0)
    CKE(cudaMalloc(&s->d_p, (N + 4) * sizeof(float)));
    CKE(cudaMalloc(&s->d_y, N * sizeof(float)));
    CKE(cudaMalloc(&s->d_z[0], (N + 4) * sizeof(float)));   // +4: 16-byte bulk copies of x
    CKE(cudaMalloc(&s->d_z[1], (N + 4) * sizeof(float)));
    CKE(cudaMemset(s->d_z[0], 0, (N + 4) * sizeof(float)));
    CKE(cudaMemset(s->d_z[1], 0, (N + 4) * sizeof(float)));
    CKE(cudaMalloc(&s->d_inv, N * sizeof(float)));
    CKE(cudaMemcpy(s->d_inv, invd_pi.data(), N * sizeof(float), cudaMemcpyHostToDevice));
    CKE(cudaMalloc(&s->d_half, std::max<int64_t>(N, 1)));
    if (!half_pi.empty()) CKE(cudaMemcpy(s->d_half, half_pi.data(), N, cudaMemcpyHostToDevice));
    CKE(cudaMalloc(&s->d_ctrl, sizeof(Ctrl)));
    CKE(cudaMemset(s->d_ctrl, 0, sizeof(Ctrl)));
    // launches and partial slots
    if (p->two_phase) {             // one persistent two-phase launch per SpMV (pb.h)
        int g = 0;
        if (s->algo == SPMV_ALGO_HITS) CKE(pb_setup<EpiHitsSpmv>(*p, g));
        else CKE(pb_setup<EpiAffine>(*p, g));
        s->grids.assign(1, g);
    } else if (s->algo == SPMV_ALGO_HITS) CKE(setup_grids<EpiHitsSpmv>(*p, s->grids));
    else CKE(setup_grids<EpiAffine>(*p, s->grids));
    s->tiles_used.clear();
    s->slot_base.clear();
    int32_t slots = 0;
    for (int32_t t = 0; t <= p->num_tiles; ++t) {
        if (!p->two_phase && p->tiles[t].wl_end == p->tiles[t].wl_begin) continue;
        s->tiles_used.push_back(t);
        s->slot_base.push_back(slots);
        slots += s->grids[t];
    }
    s->total_slots = slots;
    s->norm_grid = p->sm_count * 4;
    CKE(cudaMalloc(&s->d_slots, (size_t)std::max(slots, s->norm_grid) * 2 * sizeof(double)));
    // entry-ordered epilogue state
    std::vector<uint32_t> entries;
    if ((st = plan_final_positions(p, entries, s->fpos))) return st;
    const int64_t ne = std::max<int64_t>(p->n_row_entries, 1);
    std::vector<float> inv_e(ne, 0.0f);
    std::vector<uint8_t> half_e(ne, 0);
    for (int64_t k = 0; k < p->n_row_entries; ++k) {
        const uint32_t ent = entries[k];
        if (ent == PAD_ROW || !(ent & FLAG_FINAL)) continue;
        const uint32_t r = ent & ROW_MASK;
        inv_e[k] = invd_pi[r];
        if (!half_pi.empty()) half_e[k] = half_pi[r];
    }
    CKE(cudaMalloc(&s->d_p_e, ne * sizeof(float)));
    CKE(cudaMalloc(&s->d_inv_e, ne * sizeof(float)));
    CKE(cudaMemcpy(s->d_inv_e, inv_e.data(), ne * sizeof(float), cudaMemcpyHostToDevice));
    CKE(cudaMalloc(&s->d_half_e, ne));
    CKE(cudaMemcpy(s->d_half_e, half_e.data(), ne, cudaMemcpyHostToDevice));
    CKE(cudaMalloc(&s->d_fpos, std::max<int64_t>(N, 1) * sizeof(int32_t)));
    CKE(cudaMemcpy(s->d_fpos, s->fpos.data(), N * sizeof(int32_t), cudaMemcpyHostToDevice));
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
            epi.y = s->d_y; epi.half = s->d_half_e; epi.fpos = s->d_fpos; epi.ctrl = s->d_ctrl; epi.slots = s->d_slots;
            epi.slot_base = s->slot_base[i]; epi.total_slots = s->total_slots;
            epi.is_last = (i + 1 == nu); epi.l2 = s->it.hits_norm != 1;
            cudaError_t e = p->two_phase ? launch_pb(*p, s->grids[0], s->d_p, epi, st)
                                         : launch_tile(*p, s->tiles_used[i], s->grids[s->tiles_used[i]], s->d_p, epi, st);
            if (e) return e;
        }
        hits_normalize<<<s->norm_grid, kThreads, 0, st>>>(s->d_y, s->d_p, s->d_half, s->N, s->d_ctrl,
                                                           s->d_slots, cond);
        return cudaGetLastError();
    }
    for (size_t i = 0; i < nu; ++i) {
        EpiAffine epi{};
        epi.y = s->d_y; epi.p = s->d_p_e; epi.z_next = s->d_z[parity ^ 1]; epi.inv_deg = s->d_inv_e;
        epi.fpos = s->d_fpos;
        epi.ctrl = s->d_ctrl; epi.slots = s->d_slots; epi.slot_base = s->slot_base[i];
        epi.total_slots = s->total_slots; epi.is_last = (i + 1 == nu); epi.cond = cond;
        epi.rwr = s->algo == SPMV_ALGO_RWR;
        cudaError_t e = p->two_phase ? launch_pb(*p, s->grids[0], s->d_z[parity], epi, st)
                                     : launch_tile(*p, s->tiles_used[i], s->grids[s->tiles_used[i]], s->d_z[parity], epi, st);
        if (e) return e;
    }
    return cudaSuccess;
}

// the iteration loop without a graph: iterations (double-buffered z) enqueued in batches of 8,
// the stop flag read after each batch; *stop = the event after the iteration that stopped
static cudaError_t run_host_loop(spmv_solver_s* s, cudaStream_t st, cudaEvent_t* stop, Ctrl* hc) {
    const int batch = 8;
    const int cap = std::max(s->it.max_iter, s->it.fixed_iters) + batch;
    cudaError_t e = cudaSuccess;
    std::vector<cudaEvent_t> ev;
    int launched = 0;
    while (!e) {
        for (int b = 0; b < batch && !e; ++b, ++launched) {
            e = enqueue_iteration(s, launched & 1, st, 0);
            cudaEvent_t v;
            cudaEventCreate(&v);
            cudaEventRecord(v, st);
            ev.push_back(v);
        }
        if (!e) e = cudaMemcpyAsync(hc, s->d_ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, st);
        if (!e) e = cudaStreamSynchronize(st);
        if (e || hc->done || launched > cap) break;
    }
    if (!e && !ev.empty()) {
        // HITS counts an iteration per normalisation pass, one per body as well
        const int64_t last = std::min<int64_t>(std::max<int64_t>(hc->iter - 1, 0), (int64_t)ev.size() - 1);
        *stop = ev[last];
        ev[last] = nullptr;
    }
    for (auto v : ev) if (v) cudaEventDestroy(v);
    return e;
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
    o->tol = 1e-6; o->max_iter = 1000; o->hits_norm = 1; o->fixed_iters = 0; o->exchange = 0;
    o->host_loop = 0;
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
spmv_status spmv_solver_create_local(int algo, int64_t n_global, int64_t n_local, const int32_t* owned_ids,
                                     const int64_t* row_ptr, const int32_t* col, const int32_t* out_degree,
                                     const spmv_iter_opts* it, const spmv_options* opt, spmv_comm comm,
                                     int device, spmv_solver* out) {
    if (!out || !comm || n_global < 1 || n_local < 0 || (n_local > 0 && (!owned_ids || !row_ptr)) ||
        (n_local > 0 && row_ptr[n_local] > 0 && !col)) {
        set_error("invalid argument"); return SPMV_EINVAL;
    }
    if (algo != SPMV_ALGO_PAGERANK && algo != SPMV_ALGO_RWR && algo != SPMV_ALGO_HITS) {
        set_error("local input: unknown algorithm"); return SPMV_EINVAL;
    }
    if (algo == SPMV_ALGO_PAGERANK && n_local > 0 && !out_degree) { set_error("PageRank needs out_degree"); return SPMV_EINVAL; }
    if (algo == SPMV_ALGO_HITS && out_degree) { set_error("HITS: out_degree must be NULL"); return SPMV_EINVAL; }
    const int64_t n_rows = algo == SPMV_ALGO_HITS ? 2 * n_global : n_global;   // HITS: block rows
    if (n_local > 0 && row_ptr[0] != 0) { set_error("row_ptr[0] != 0"); return SPMV_EINVAL; }
    for (int64_t i = 0; i < n_local; ++i) {
        if (row_ptr[i + 1] < row_ptr[i]) { set_error("row_ptr not monotone"); return SPMV_EINVAL; }
        if (owned_ids[i] < 0 || owned_ids[i] >= n_rows) { set_error("owned id out of range"); return SPMV_ERANGE; }
        if (out_degree && out_degree[i] < 0) { set_error("negative degree"); return SPMV_EINVAL; }
    }
    if (device < 0) { set_error("solvers need a device"); return SPMV_EINVAL; }
    LocalInput li{n_local, owned_ids, row_ptr, col, out_degree};
    return solver_create_dist(algo, n_global, n_local > 0 ? row_ptr[n_local] : 0, nullptr, nullptr, it, opt, comm,
                              device, out, &li);
}

__attribute__((visibility("default")))
spmv_status spmv_solver_run(spmv_solver s, int64_t query, void* stream, spmv_iter_result* res) {
    if (!s) { set_error("null solver"); return SPMV_EINVAL; }
    if (s->comm) return solver_run_dist(s, query, stream, res);
    Range r_run("spmv_solver_run");
    if (s->algo == SPMV_ALGO_RWR && (query < 0 || query >= s->n)) { set_error("query out of range"); return SPMV_ERANGE; }
    cudaError_t e = cudaSetDevice(s->device);
    if (e) return cuda_status(e, "cudaSetDevice");
    cudaStream_t st = (cudaStream_t)stream;
    if (!st) {
        if (!s->own_stream && (e = cudaStreamCreateWithFlags(&s->own_stream, cudaStreamNonBlocking)))
            return cuda_status(e, "stream");
        st = s->own_stream;
    }
    if (!s->exec && !s->it.host_loop) { spmv_status b = build_graph(s, st); if (b) return b; }
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
    else {
        init_affine<<<g, 256, 0, st>>>(s->d_p, s->d_z[0], s->d_inv, s->N, s->algo == SPMV_ALGO_RWR,
                                       (int32_t)c.q, (float)(1.0 / n));
        init_entries<<<g, 256, 0, st>>>(s->d_p_e, s->plan->d_row_id, s->plan->n_row_entries,
                                        s->algo == SPMV_ALGO_RWR, (int32_t)c.q, (float)(1.0 / n));
    }
    if ((e = cudaGetLastError())) return cuda_status(e, "init");
    Ctrl* hc = nullptr;                       // pinned, allocated before the timed region
    if (s->it.host_loop && (e = cudaMallocHost(&hc, sizeof(Ctrl)))) return cuda_status(e, "cudaMallocHost");
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0, st);
    cudaEvent_t e_stop = nullptr;
    if (s->it.host_loop) e = run_host_loop(s, st, &e_stop, hc);   // the same kernels, host-enqueued
    else e = cudaGraphLaunch(s->exec, st);
    if (hc) cudaFreeHost(hc);
    cudaEventRecord(e1, st);
    if (e) {
        cudaEventDestroy(e0); cudaEventDestroy(e1);
        if (e_stop) cudaEventDestroy(e_stop);
        return cuda_status(e, "iteration loop");
    }
    if ((e = cudaMemcpyAsync(&c, s->d_ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, st)) ||
        (e = cudaStreamSynchronize(st))) {
        cudaEventDestroy(e0); cudaEventDestroy(e1);
        if (e_stop) cudaEventDestroy(e_stop);
        return cuda_status(e, "iteration loop");
    }
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e_stop ? e_stop : e1);
    cudaEventDestroy(e0); cudaEventDestroy(e1);
    if (e_stop) cudaEventDestroy(e_stop);
    s->last = c;
    if (res) {
        res->iterations = c.iter; res->residual = c.residual;
        res->converged = s->it.fixed_iters > 0 ? 1 : (c.residual < s->it.tol);
        res->ms_total = ms; res->us_per_iter = c.iter ? 1000.0 * ms / c.iter : 0.0;
        res->predicted_us_per_iter = s->plan->predicted_us + s->pred_extra_us;
        res->phase_us[0] = res->us_per_iter; res->phase_us[1] = res->phase_us[2] = 0.0;
    }
    if (s->it.fixed_iters <= 0 && !(c.residual < s->it.tol)) { set_error("max_iter reached"); return SPMV_ENOCONV; }
    return SPMV_OK;
}

__attribute__((visibility("default")))
spmv_status spmv_solver_result(spmv_solver s, float* out0, float* out1) {
    if (!s || !out0 || (s->algo == SPMV_ALGO_HITS && !out1)) { set_error("null argument"); return SPMV_EINVAL; }
    if (s->comm) return solver_result_dist(s, out0, out1);
    cudaSetDevice(s->device);
    std::vector<float> v(s->N);
    cudaError_t e;
    if (s->algo == SPMV_ALGO_HITS) {
        e = cudaMemcpy(v.data(), s->d_p, s->N * sizeof(float), cudaMemcpyDeviceToHost);
    } else {   // PageRank / RWR keep p in row-entry order
        std::vector<float> pe(std::max<int64_t>(s->plan->n_row_entries, 1));
        e = cudaMemcpy(pe.data(), s->d_p_e, s->plan->n_row_entries * sizeof(float), cudaMemcpyDeviceToHost);
        for (int64_t r = 0; r < s->N; ++r) v[r] = s->fpos[r] >= 0 ? pe[s->fpos[r]] : 0.0f;
    }
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

__attribute__((visibility("default")))
spmv_status spmv_solver_set_stop(spmv_solver s, double tol, int32_t max_iter, int32_t fixed_iters) {
    if (!s || !(tol >= 0.0) || max_iter < 1 || fixed_iters < 0) { set_error("invalid argument"); return SPMV_EINVAL; }
    s->it.tol = tol; s->it.max_iter = max_iter; s->it.fixed_iters = fixed_iters;   // read per run (Ctrl)
    return SPMV_OK;
}

__attribute__((visibility("default"))) int32_t spmv_solver_launches_per_iter(spmv_solver s) {
    if (!s) return 0;
    return (int32_t)s->tiles_used.size() + (s->algo == SPMV_ALGO_HITS ? 1 : 0);
}

__attribute__((visibility("default"))) void spmv_solver_destroy(spmv_solver s) {
    if (!s) return;
    if (s->comm) { solver_destroy_dist(s); return; }
    cudaSetDevice(s->device);
    batch_destroy(s);
    if (s->exec) cudaGraphExecDestroy(s->exec);
    if (s->graph) cudaGraphDestroy(s->graph);
    if (s->own_stream) cudaStreamDestroy(s->own_stream);
    cudaFree(s->d_p); cudaFree(s->d_y); cudaFree(s->d_z[0]); cudaFree(s->d_z[1]); cudaFree(s->d_inv);
    cudaFree(s->d_half); cudaFree(s->d_ctrl); cudaFree(s->d_slots);
    cudaFree(s->d_p_e); cudaFree(s->d_inv_e); cudaFree(s->d_half_e); cudaFree(s->d_fpos);
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
