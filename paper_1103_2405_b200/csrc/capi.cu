// capi.cu -- C ABI: plan creation, upload, spmv_execute (include/spmv.h).
#include <cstdio>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <string>

#include "launch.cuh"
#include "pb_launch.cuh"

#ifndef TC_PDL
#define TC_PDL 1          // experiment builds: -DTC_PDL=0 launches every tile plainly (bench/explore_pdl.py)
#endif

#include "trace.h"
#include "tune.h"

namespace tc {

static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }
spmv_status cuda_status(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return SPMV_OK;
    set_error(std::string(what) + ": " + cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? SPMV_ENOMEM : SPMV_ECUDA;
}

// xp[k] = x[perm[k]] (step a7): relabel x for the tiled product
__global__ void permute_x_kernel(const float* __restrict__ x, const int32_t* __restrict__ perm,
                                 float* __restrict__ xp, int64_t n) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    asm volatile("griddepcontrol.launch_dependents;");   // tile 0 may launch (it waits for us)
    for (; i < n; i += stride) xp[i] = __ldg(x + __ldcs(perm + i));
}

// x'[inv[j]] = x[j]: x and inv read coalesced (16-byte vectors), x' written by scattered 4-byte
// stores, which need no response (the gather form waits on 4.85 M random reads on c2)
__global__ void scatter_x_kernel(const float* __restrict__ x, const int32_t* __restrict__ inv,
                                 float* __restrict__ xp, int64_t n) {
    const int64_t n4 = n >> 2;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const float4* x4 = reinterpret_cast<const float4*>(x);
    const int4* i4 = reinterpret_cast<const int4*>(inv);
    const bool vec = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(inv)) & 15) == 0;
    asm volatile("griddepcontrol.launch_dependents;");   // tile 0 may launch (it waits for us)
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (vec) {
        for (; i < n4; i += stride) {
            const float4 v = __ldcs(x4 + i);
            const int4 k = __ldcs(i4 + i);
            xp[k.x] = v.x; xp[k.y] = v.y; xp[k.z] = v.z; xp[k.w] = v.w;
        }
        for (int64_t j = 4 * n4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride) xp[inv[j]] = x[j];
    } else {
        for (; i < n; i += stride) xp[__ldcs(inv + i)] = __ldcs(x + i);
    }
}

template <class T>
static cudaError_t upload(T** dst, const std::vector<T>& src, int64_t& bytes) {
    size_t nb = std::max<size_t>(src.size(), 1) * sizeof(T);
    cudaError_t e = cudaMalloc(dst, nb);
    if (e) return e;
    bytes += (int64_t)nb;
    if (!src.empty()) e = cudaMemcpy(*dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice);
    return e;
}

template <class T>
static cudaError_t download(std::vector<T>& dst, const T* src, int64_t n) {
    dst.resize(n);
    if (n == 0) return cudaSuccess;
    return cudaMemcpy(dst.data(), src, n * sizeof(T), cudaMemcpyDeviceToHost);
}

static std::vector<int32_t> inverse(const std::vector<int32_t>& perm) {
    std::vector<int32_t> inv(perm.size());
    for (size_t k = 0; k < perm.size(); ++k) inv[perm[k]] = (int32_t)k;
    return inv;
}

// x' = x relabelled (a7): gather form by default; TCSPMV_PERMUTE=scatter selects the scatter form
// (measured on c2: 354 vs 352 us per SpMV, profiles/r01_permute_forms.jsonl)
static cudaError_t launch_permute(spmv_plan_s* p, const float* x, cudaStream_t st) {
    int grid = (int)std::min<int64_t>((p->n_cols + 255) / 256, (int64_t)p->sm_count * 8);
    if (p->permute_gather) permute_x_kernel<<<grid, 256, 0, st>>>(x, p->d_perm, p->d_xp, p->n_cols);
    else scatter_x_kernel<<<grid, 256, 0, st>>>(x, p->d_inv, p->d_xp, p->n_cols);
    return cudaGetLastError();
}

static void free_device(spmv_plan_s* p) {
    if (p->device < 0) return;
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(p->device);
    cudaFree(p->d_desc); cudaFree(p->d_row_id); cudaFree(p->d_col); cudaFree(p->d_val);
    cudaFree(p->d_perm); cudaFree(p->d_inv); cudaFree(p->d_xp); cudaFree(p->d_split); cudaFree(p->d_partials);
    cudaFree(p->d_counters); cudaFree(p->d_hx); cudaFree(p->d_sched); cudaFree(p->d_hxb);
    cudaFree(p->d_pb_runs); cudaFree(p->d_pb_cd);
    cudaFree(p->d_pb_val); cudaFree(p->d_pb_pos); cudaFree(p->d_pb_pmeta); cudaFree(p->d_pb_items);
    cudaFree(p->d_pb_gchunks); cudaFree(p->d_pb_buf); cudaFree(p->d_pb_ctl);
    if (p->s_h2d) cudaStreamDestroy(p->s_h2d);
    if (p->s_d2h) cudaStreamDestroy(p->s_d2h);
    for (auto& ev : p->ev_pipe) if (ev) cudaEventDestroy(ev);
    if (p->ev_scratch) cudaEventDestroy(p->ev_scratch);
    cudaSetDevice(cur);
}

// the device work queue: descriptors in queue order
static std::vector<PbItem> pb_queue(const PbLayout& B) {
    std::vector<PbItem> q(B.items.size());
    for (size_t i = 0; i < B.items.size(); ++i) {
        PbItem& t = q[i];
        const int32_t code = B.items[i];
        if (code >= 0) {
            const PbChunk& c = B.chunks[code];
            t.a0 = c.e0; t.a1 = c.gbase; t.a2 = c.run0; t.n = c.n; t.b0 = c.col0; t.b1 = c.span; t.b2 = c.nrun;
            t.group = c.group; t.kind = PB_ITEM_EXPAND;
        } else {
            const PbBin& b = B.bins[~code];
            t.a0 = b.roff; t.a1 = b.poff; t.a2 = b.row0; t.n = b.rlen; t.b0 = b.plen; t.b1 = b.nrows; t.b2 = b.nheavy;
            t.group = b.group; t.kind = b.kind == PB_LONG ? PB_ITEM_LONG : PB_ITEM_BIN;
        }
    }
    if (q.empty()) q.push_back(PbItem{});
    return q;
}

// Two-phase plan (pb.h): layout over the original row and column ids (no relabel of x: the chunks
// stage whatever columns they cover), uploaded with its partial buffer and queue counters.
static spmv_status create_two_phase(spmv_plan_s* p, const Prepared& P, const int64_t* row_ptr,
                                    const int32_t* col, const float* val, const PbParams& prm,
                                    std::chrono::steady_clock::time_point t0, bool built) {
    if (!built && !pb_build_fit(p->n_rows, p->n_cols, row_ptr, col, p->pattern ? nullptr : val, p->pattern, prm,
                                p->opt.pb_xcap > 0, p->PB)) {
        delete p; return SPMV_EINVAL;
    }
    PbLayout& B = p->PB;
    if (!built) p->two_phase_us = pb_predict_items_us(p->opt, (int64_t)B.items.size(), !p->pattern);
    p->perm.resize(p->n_cols);
    for (int64_t k = 0; k < p->n_cols; ++k) p->perm[k] = (int32_t)k;
    (void)P;
    p->num_tiles = 0; p->tile_width = (int32_t)std::min<int64_t>(p->n_cols, INT32_MAX);
    p->tiles.assign(1, TileInfo{});
    p->tiles[0].col_hi = p->n_cols; p->tiles[0].nnz = p->nnz; p->tiles[0].rows = p->n_rows;
    p->tiles[0].pred_us = p->two_phase_us;
    p->predicted_us = p->two_phase_us;
    p->n_row_entries = p->n_rows;
    p->pb_chunks = (int64_t)B.chunks.size(); p->pb_bins = (int64_t)B.bins.size(); p->pb_groups = B.n_groups;
    for (auto& b : B.bins) p->pb_long += b.kind == PB_LONG;
    p->pb_smem = kPbStages * B.stage_bytes;
    if (p->pb_smem > 227 * 1024) { delete p; set_error("two-phase stage exceeds shared memory"); return SPMV_EINVAL; }
    p->L.row_id = B.prow;
    p->host_valid = true;
    p->pb_host_valid = true;
    if (p->device >= 0) {
        cudaError_t e;
        int64_t& b = p->device_bytes;
        std::vector<float> zbuf;
        std::vector<uint32_t> zctl(2 + std::max(B.n_groups, 1), 0u);
        // streams copied in 16-byte granules from a 16-byte boundary: 4 elements of tail padding
        for (int i = 0; i < 4; ++i) {
            B.runs.push_back(0); B.cd.push_back(0u); B.prow.push_back(PAD_ROW); B.pmeta.push_back(0u);
            if (!p->pattern) B.val.push_back(0.0f);
        }
        if ((e = upload(&p->d_pb_runs, B.runs, b)) || (e = upload(&p->d_pb_cd, B.cd, b)) ||
            (!p->pattern && (e = upload(&p->d_pb_val, B.val, b))) || (e = upload(&p->d_pb_pos, B.pos, b)) ||
            (e = upload(&p->d_row_id, B.prow, b)) || (e = upload(&p->d_pb_pmeta, B.pmeta, b)) ||
            (e = upload(&p->d_pb_items, pb_queue(B), b)) || (e = upload(&p->d_pb_gchunks, B.group_chunks, b)) ||
            (e = upload(&p->d_pb_ctl, zctl, b))) {
            free_device(p); delete p; return cuda_status(e, "two-phase upload");
        }
        if ((e = cudaMalloc(&p->d_pb_buf, (size_t)B.buf_floats * sizeof(float)))) {
            free_device(p); delete p; return cuda_status(e, "two-phase buffer");
        }
        b += B.buf_floats * (int64_t)sizeof(float);
        std::vector<float> xpz(p->n_cols + 4, 0.0f);
        if ((e = upload(&p->d_xp, xpz, b))) { free_device(p); delete p; return cuda_status(e, "plan upload"); }
        if ((e = pb_setup<EpiStore>(*p, p->pb_grid))) { free_device(p); delete p; return cuda_status(e, "occupancy"); }
        // the per-entry arrays live on the device (fetched back on demand by to_coo)
        B.cd = {}; B.val = {}; B.pos = {}; B.prow = {}; B.pmeta = {}; B.runs = {};
        p->L.row_id = {};
        p->host_valid = false;
        p->pb_host_valid = false;
    }
    p->build_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    return SPMV_OK;
}

// Upload a one-pass plan's host layout to p->device (plan creation and spmv_plan_import); on
// failure the plan is freed.
static spmv_status upload_one_pass(spmv_plan_s* p) {
    cudaError_t e;
    int64_t& b = p->device_bytes;
    if (const char* h = std::getenv("TCSPMV_PERMUTE")) p->permute_gather = std::string(h) != "scatter";
    if ((e = upload(&p->d_desc, p->L.desc, b)) || (e = upload(&p->d_row_id, p->L.row_id, b)) ||
        (e = upload(&p->d_col, p->L.slot_col, b)) || (e = upload(&p->d_perm, p->perm, b)) ||
        (!p->permute_gather && (e = upload(&p->d_inv, inverse(p->perm), b))) ||
        (e = upload(&p->d_split, p->L.split, b))) {
        free_device(p); delete p; return cuda_status(e, "plan upload");
    }
    if (!p->pattern && (e = upload(&p->d_val, p->L.slot_val, b))) {
        free_device(p); delete p; return cuda_status(e, "plan upload");
    }
    std::vector<float> zf(std::max<int64_t>(p->n_chunks, 1), 0.0f);
    std::vector<int32_t> zi(std::max<int64_t>(p->n_split, 1), 0);
    std::vector<float> xpz(p->n_cols + 4, 0.0f);
    std::vector<uint32_t> zs((size_t)(tc::kDynQ + 1) * (p->num_tiles + 1), 0u);
    if ((e = upload(&p->d_partials, zf, b)) || (e = upload(&p->d_counters, zi, b)) ||
        (e = upload(&p->d_sched, zs, b)) ||
        (e = upload(&p->d_xp, xpz, b))) {
        free_device(p); delete p; return cuda_status(e, "plan upload");
    }
    if ((e = setup_grids<EpiStore>(*p, p->grid_tile))) {
        free_device(p); delete p; return cuda_status(e, "occupancy");
    }
    // release the host copy (fetched back on demand by spmv_plan_layout / to_coo)
    p->L.desc = {}; p->L.row_id = {}; p->L.slot_col = {}; p->L.slot_val = {}; p->L.split = {};
    p->host_valid = false;
    return SPMV_OK;
}

// build the plan (host) and upload it; shared by spmv_plan_create and the solvers
spmv_status create_plan(int64_t n_rows, int64_t n_cols, int64_t nnz, const int64_t* row_ptr,
                        const int32_t* col, const float* val, const spmv_options* opt_in,
                        int device, spmv_plan_s** out) {
    auto t0 = std::chrono::steady_clock::now();
    spmv_options opt;
    if (opt_in) opt = *opt_in; else spmv_options_default(&opt);
    if (opt.orient < -1 || opt.orient > 3) { set_error("orient must be -1, 0, 1, 2 or 3"); return SPMV_EINVAL; }
    if (device >= 0 && (opt.ell_h != 32 || opt.align_rm % 4 != 0)) {
        set_error("device plans need ell_h = 32 and align_rm % 4 == 0"); return SPMV_EINVAL;
    }
    int sm_count = 148;
    if (device >= 0) {
        int ndev = 0;
        cudaError_t e = cudaGetDeviceCount(&ndev);
        if (e != cudaSuccess || ndev == 0) { set_error("no CUDA device"); return SPMV_ECUDA; }
        if (device >= ndev) { set_error("device ordinal out of range"); return SPMV_EINVAL; }
        if ((e = cudaSetDevice(device))) return cuda_status(e, "cudaSetDevice");
        cudaDeviceGetAttribute(&sm_count, cudaDevAttrMultiProcessorCount, device);
    }
    Range r_build("spmv_plan_create");
    Prepared P;
    if (opt.keep_col_order && opt.two_phase == 1) { set_error("keep_col_order is a one-pass option"); return SPMV_EINVAL; }
    spmv_status st = prepare(n_rows, n_cols, nnz, row_ptr, col, val, opt.pattern != 0, P, opt.keep_col_order != 0);
    if (st) return st;
    BuildParams bp;
    std::vector<double> pred;
    int32_t table_loaded = 0;
    {
        Range r("tune (Alg. 1-3)");
        st = choose_params(P, opt, sm_count, bp, pred, &table_loaded);
    }
    if (st) return st;
    if (opt.two_phase < -1 || opt.two_phase > 1) { set_error("two_phase must be -1, 0 or 1"); return SPMV_EINVAL; }
    spmv_plan_s* p = new spmv_plan_s();
    p->n_rows = n_rows; p->n_cols = n_cols; p->nnz = nnz; p->pattern = opt.pattern != 0;
    p->device = device; p->opt = opt; p->sm_count = sm_count; p->perf_table_loaded = table_loaded;
    p->opt.workload_sizes = nullptr; p->opt.perf_table_path = nullptr;
    // one-pass tiles (Alg. 1-3) or two-phase tiles: the model's choice unless forced
    const PbParams prm = pb_params(opt, n_cols, nnz);
    for (double u : pred) p->one_pass_us += u;
    p->two_phase_us = pb_predict_us(opt, n_rows, n_cols, nnz, opt.pattern == 0, prm);
    // in auto mode an explicit one-pass parameter (tile width / count, WL, orientation, paper mode)
    // asks for the one-pass tiles
    const bool one_pass_forced = opt.tile_width > 0 || opt.num_tiles >= 0 || opt.workload_size > 0 ||
                                 opt.workload_sizes || opt.orient != 0 || opt.split_long_rows == 0 ||
                                 opt.keep_col_order != 0;
    p->two_phase = opt.two_phase == 1;
    bool built = false;
    if (opt.two_phase == -1 && !one_pass_forced && nnz > 0 && p->two_phase_us < 1.25 * p->one_pass_us) {
        // close enough to matter: build the layout and predict from its actual item count
        if (pb_build_fit(n_rows, n_cols, row_ptr, col, p->pattern ? nullptr : val, p->pattern, prm, opt.pb_xcap > 0,
                         p->PB)) {
            built = true;
            p->two_phase_us = pb_predict_items_us(opt, (int64_t)p->PB.items.size(), !p->pattern);
            p->two_phase = p->two_phase_us < p->one_pass_us;
        }
        if (!p->two_phase) p->PB = PbLayout();
    }
    if (p->two_phase) {
        st = create_two_phase(p, P, row_ptr, col, val, prm, t0, built);
        if (!st) *out = p;
        return st;
    }
    {
        Range r("pack_layout");
        p->orient = bp.orient;
    st = pack_layout(P, bp, p->L);
    }
    if (st) { delete p; return st; }
    p->perm = std::move(P.perm);
    p->host_valid = true;
    p->num_tiles = bp.num_tiles; p->tile_width = bp.tile_width;
    p->tiles = p->L.tiles;
    p->n_workloads = (int64_t)p->L.desc.size();
    p->n_slots = (int64_t)p->L.slot_col.size();
    p->n_row_entries = (int64_t)p->L.row_id.size();
    p->n_split = (int64_t)p->L.split.size() / 3;
    p->n_chunks = p->L.n_chunks;
    predict_plan(*p, pred);
    // programmatic dependent launch between the standalone launches when they are short enough for
    // the ~5 us launch gap to matter (measured, profiles/r02_pdl.log: 8 tiles of 16K columns on c2
    // -3 %, c3 youtube 4 tiles -10 %; two 48K tiles on c2 +2.6 %, c4's 1 ms launches +0.8 %)
    {
        const int32_t nl = spmv_plan_launches(p);
        p->pdl = TC_PDL && nl > 1 && p->predicted_us / nl < 64.0;
    }
    for (int32_t t = 0; t < p->num_tiles; ++t)
        p->tiles[t].staged = (opt.stage_x != 0) && (p->tiles[t].col_hi - p->tiles[t].col_lo) * 4 <= 227 * 1024 &&
                             (p->tiles[t].col_lo % 4 == 0);
    if (device >= 0 && (st = upload_one_pass(p))) return st;
    p->build_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    *out = p;
    return SPMV_OK;
}

static spmv_status ensure_host(spmv_plan_s* p) {
    if (p->host_valid) return SPMV_OK;
    cudaSetDevice(p->device);
    cudaError_t e;
    if ((e = download(p->L.desc, p->d_desc, p->n_workloads)) ||
        (e = download(p->L.row_id, p->d_row_id, p->n_row_entries)) ||
        (e = download(p->L.slot_col, p->d_col, p->n_slots)) ||
        (e = download(p->L.split, p->d_split, 3 * p->n_split)))
        return cuda_status(e, "layout download");
    if (!p->pattern && (e = download(p->L.slot_val, p->d_val, p->n_slots)))
        return cuda_status(e, "layout download");
    p->host_valid = true;
    return SPMV_OK;
}

// two-phase layout arrays back on the host (released after upload)
static spmv_status pb_ensure_host(spmv_plan_s* p) {
    if (p->pb_host_valid) return SPMV_OK;
    cudaSetDevice(p->device);
    PbLayout& B = p->PB;
    int64_t nruns = 0, npos = 0;
    for (auto& c : B.chunks) nruns = std::max<int64_t>(nruns, c.run0 + c.nrun);
    for (auto& b : B.bins) npos = std::max<int64_t>(npos, b.poff + b.plen);
    cudaError_t e;
    if ((e = download(B.cd, p->d_pb_cd, p->nnz)) || (e = download(B.pos, p->d_pb_pos, npos)) ||
        (e = download(B.prow, p->d_row_id, p->n_rows)) || (e = download(B.pmeta, p->d_pb_pmeta, p->n_rows)) ||
        (e = download(B.runs, p->d_pb_runs, std::max<int64_t>(nruns, 1))) ||
        (!p->pattern && (e = download(B.val, p->d_pb_val, p->nnz))))
        return cuda_status(e, "two-phase layout download");
    p->pb_host_valid = true;
    return SPMV_OK;
}

// Decode the two-phase layout to COO: the expand's destination of every entry, then the reduce's
// positions of every row (checks that every entry lands in exactly one row's list).
static spmv_status pb_to_coo(spmv_plan_s* p, int32_t* rows, int32_t* cols, float* vals) {
    spmv_status s = pb_ensure_host(p);
    if (s) return s;
    const PbLayout& B = p->PB;
    std::vector<int64_t> src(B.buf_floats, -1);
    std::vector<int32_t> ecol(p->nnz);
    for (const PbChunk& c : B.chunks)
        for (int32_t k = 0; k < c.n; ++k) {
            const int64_t e = c.e0 + k;
            const uint32_t w = B.cd[e];
            const int64_t idx = c.gbase + k + B.runs[c.run0 + (w >> 16)];
            if (idx < 0 || idx >= B.buf_floats || src[idx] >= 0) { set_error("two-phase destinations overlap"); return SPMV_EINVAL; }
            src[idx] = e;
            ecol[e] = c.col0 + (int32_t)(w & 0xffffu);
        }
    int64_t out = 0;
    std::vector<uint8_t> seen(p->nnz, 0);
    auto put = [&](uint32_t ent, int64_t idx) -> bool {
        const int64_t e = idx >= 0 && idx < B.buf_floats ? src[idx] : -1;
        if (e < 0 || seen[e] || out >= p->nnz) return false;
        seen[e] = 1;
        rows[out] = (int32_t)(ent & ROW_MASK);
        cols[out] = ecol[e];
        if (vals) vals[out] = p->pattern ? 1.0f : B.val[e];
        ++out;
        return true;
    };
    for (const PbBin& b : B.bins) {
        if (b.kind == PB_LONG) {
            for (int32_t q = 0; q < b.rlen; ++q)
                if (!put(B.prow[b.row0], b.roff + q)) { set_error("two-phase decode"); return SPMV_EINVAL; }
            continue;
        }
        for (int32_t r = 0; r < b.nrows; ++r) {
            const uint32_t m = B.pmeta[b.row0 + r];
            const int64_t po = m & 0xffffu, ln = m >> 16, stride = r < b.nheavy ? 1 : 32;
            for (int64_t t = 0; t < ln; ++t)
                if (!put(B.prow[b.row0 + r], b.roff + B.pos[b.poff + po + stride * t])) {
                    set_error("two-phase decode"); return SPMV_EINVAL;
                }
        }
    }
    if (out != p->nnz) { set_error("two-phase decode count mismatch"); return SPMV_EINVAL; }
    return SPMV_OK;
}

// Row-entry bookkeeping for entry-ordered epilogue state: the row entries (host copy) and, per
// row, the index of its FINAL entry (the first one for split rows); -1 for rows without one.
spmv_status plan_final_positions(spmv_plan_s* p, std::vector<uint32_t>& entries, std::vector<int32_t>& fpos) {
    entries.resize(p->n_row_entries);
    if (p->host_valid) entries = p->L.row_id;
    else if (p->n_row_entries) {
        cudaError_t e = cudaMemcpy(entries.data(), p->d_row_id, p->n_row_entries * sizeof(uint32_t), cudaMemcpyDeviceToHost);
        if (e) return cuda_status(e, "row entries");
    }
    fpos.assign(p->n_rows, -1);
    for (int64_t k = 0; k < p->n_row_entries; ++k) {
        const uint32_t ent = entries[k];
        if (ent == PAD_ROW || !(ent & FLAG_FINAL)) continue;
        int32_t& f = fpos[ent & ROW_MASK];
        if (f < 0) f = (int32_t)k;
    }
    return SPMV_OK;
}

// Serialise products that share the plan's scratch across streams: wait for the
// previous product when it ran on another stream; record the end of this one.
static cudaError_t scratch_acquire(spmv_plan_s* p, cudaStream_t st) {
    cudaError_t e = cudaSuccess;
    if (!p->ev_scratch && (e = cudaEventCreateWithFlags(&p->ev_scratch, cudaEventDisableTiming))) return e;
    if (p->scratch_used && p->scratch_stream != st) e = cudaStreamWaitEvent(st, p->ev_scratch, 0);
    return e;
}
static cudaError_t scratch_release(spmv_plan_s* p, cudaStream_t st) {
    cudaError_t e = cudaEventRecord(p->ev_scratch, st);
    p->scratch_stream = st;
    p->scratch_used = true;
    return e;
}

// the bulk copies of x segments need a 16-byte aligned x (else a copy in the plan's buffer)
static const float* pb_x(spmv_plan_s* p, const float* x, cudaStream_t st, cudaError_t& e) {
    e = cudaSuccess;
    if (!(reinterpret_cast<uintptr_t>(x) & 15)) return x;
    e = cudaMemcpyAsync(p->d_xp, x, p->n_cols * sizeof(float), cudaMemcpyDeviceToDevice, st);
    return p->d_xp;
}

spmv_status execute_permuted(spmv_plan_s* p, const float* xp, float* y, cudaStream_t st) {
    Range r("spmv_execute");
    if (p->two_phase) {
        cudaError_t e;
        xp = pb_x(p, xp, st, e);
        if (e) return cuda_status(e, "x alignment copy");
        return cuda_status(launch_pb(*p, p->pb_grid, xp, EpiStore{y}, st), "two-phase launch");
    }
    return cuda_status(launch_tiles(*p, p->grid_tile, xp, EpiStore{y}, st, p->pdl), "tile launch");
}

}  // namespace tc

using namespace tc;

extern "C" {

__attribute__((visibility("default"))) void spmv_options_default(spmv_options* o) {
    if (!o) return;
    std::memset(o, 0, sizeof(*o));
    o->tile_width = 0; o->num_tiles = -1; o->workload_size = -1; o->workload_sizes = nullptr;
    o->align_rm = 8; o->split_long_rows = 1; o->camping_pad = 0; o->pattern = 0; o->ell_h = 32;
    o->stage_x = 1; o->perf_table_path = nullptr; o->orient = 0;
    o->two_phase = -1; o->pb_region = 0; o->pb_chunk = 0; o->pb_xcap = 0; o->pb_group = 0;
    o->keep_col_order = 0;
}

__attribute__((visibility("default")))
spmv_status spmv_plan_create(int64_t n_rows, int64_t n_cols, int64_t nnz, const int64_t* row_ptr,
                             const int32_t* col_idx, const float* val, const spmv_options* opt,
                             int device, spmv_plan* out) {
    if (!out) { set_error("out is NULL"); return SPMV_EINVAL; }
    *out = nullptr;
    try {
        return create_plan(n_rows, n_cols, nnz, row_ptr, col_idx, val, opt, device, out);
    } catch (const std::bad_alloc&) {
        set_error("host allocation failed"); return SPMV_ENOMEM;
    } catch (const std::exception& ex) {
        set_error(ex.what()); return SPMV_EINVAL;
    }
}

__attribute__((visibility("default"))) void spmv_plan_destroy(spmv_plan p) {
    if (!p) return;
    free_device(p);
    delete p;
}

__attribute__((visibility("default")))
spmv_status spmv_execute_permuted(spmv_plan p, const float* xp, float* y, void* stream) {
    if (!p || !xp || !y) { set_error("null argument"); return SPMV_EINVAL; }
    if (p->device < 0) { set_error("host-only plan cannot execute"); return SPMV_EINVAL; }
    cudaError_t e = cudaSetDevice(p->device);
    if (e) return cuda_status(e, "cudaSetDevice");
    cudaStream_t st = (cudaStream_t)stream;
    if ((e = scratch_acquire(p, st))) return cuda_status(e, "scratch order");
    spmv_status s = execute_permuted(p, xp, y, st);
    if ((e = scratch_release(p, st)) && !s) s = cuda_status(e, "scratch order");
    return s;
}

__attribute__((visibility("default")))
spmv_status spmv_execute(spmv_plan p, const float* x, float* y, void* stream) {
    if (!p || !x || !y) { set_error("null argument"); return SPMV_EINVAL; }
    if (p->device < 0) { set_error("host-only plan cannot execute"); return SPMV_EINVAL; }
    cudaError_t e = cudaSetDevice(p->device);
    if (e) return cuda_status(e, "cudaSetDevice");
    cudaStream_t st = (cudaStream_t)stream;
    if ((e = scratch_acquire(p, st))) return cuda_status(e, "scratch order");
    spmv_status s = SPMV_OK;
    if (p->two_phase) s = execute_permuted(p, x, y, st);    // no relabel of x (pb.h)
    else {
        if (p->n_cols > 0 && (e = launch_permute(p, x, st))) s = cuda_status(e, "permute_x");
        if (!s) s = execute_permuted(p, p->d_xp, y, st);
    }
    if ((e = scratch_release(p, st)) && !s) s = cuda_status(e, "scratch order");
    return s;
}

__attribute__((visibility("default")))
spmv_status spmv_execute_host(spmv_plan p, const float* xh, float* yh, void* stream) {
    if (!p || !xh || !yh) { set_error("null argument"); return SPMV_EINVAL; }
    if (p->device < 0) { set_error("host-only plan cannot execute"); return SPMV_EINVAL; }
    cudaError_t e = cudaSetDevice(p->device);
    if (e) return cuda_status(e, "cudaSetDevice");
    cudaStream_t st = (cudaStream_t)stream;
    // device staging buffers owned by the plan (allocated on first use)
    if (!p->d_hx && (e = cudaMalloc(&p->d_hx, std::max<int64_t>(p->n_cols, 1) * 4 + std::max<int64_t>(p->n_rows, 1) * 4)))
        return cuda_status(e, "cudaMalloc");
    float* dx = p->d_hx;
    float* dy = p->d_hx + std::max<int64_t>(p->n_cols, 1);
    spmv_status s = SPMV_OK;
    if ((e = cudaMemcpyAsync(dx, xh, p->n_cols * 4, cudaMemcpyHostToDevice, st))) s = cuda_status(e, "H2D");
    if (!s) s = spmv_execute(p, dx, dy, stream);
    if (!s && (e = cudaMemcpyAsync(yh, dy, p->n_rows * 4, cudaMemcpyDeviceToHost, st))) s = cuda_status(e, "D2H");
    if (!s && (e = cudaStreamSynchronize(st))) s = cuda_status(e, "sync");
    return s;
}

__attribute__((visibility("default")))
spmv_status spmv_execute_host_batch(spmv_plan p, const float* xh, float* yh, int32_t count, void* stream) {
    if (!p || ((!xh || !yh) && count > 0) || count < 0) { set_error("null argument or count < 0"); return SPMV_EINVAL; }
    if (p->device < 0) { set_error("host-only plan cannot execute"); return SPMV_EINVAL; }
    if (count == 0) return SPMV_OK;
    cudaError_t e = cudaSetDevice(p->device);
    if (e) return cuda_status(e, "cudaSetDevice");
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t nx = std::max<int64_t>(p->n_cols, 1), ny = std::max<int64_t>(p->n_rows, 1);
    if (!p->d_hxb) {
        if ((e = cudaMalloc(&p->d_hxb, (int64_t)spmv_plan_s::kPipe * (nx + ny) * 4))) return cuda_status(e, "cudaMalloc");
        if ((e = cudaStreamCreateWithFlags(&p->s_h2d, cudaStreamNonBlocking))) return cuda_status(e, "stream");
        if ((e = cudaStreamCreateWithFlags(&p->s_d2h, cudaStreamNonBlocking))) return cuda_status(e, "stream");
        for (auto& ev : p->ev_pipe)
            if ((e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming))) return cuda_status(e, "event");
    }
    cudaEvent_t* h2d_done = p->ev_pipe;       // x buffer k filled
    const int NP = spmv_plan_s::kPipe;             // buffer pairs in use
    constexpr int KP = spmv_plan_s::kPipe;
    cudaEvent_t* comp_done = p->ev_pipe + KP;      // product on buffer pair k finished (x free, y ready)
    cudaEvent_t* d2h_done = p->ev_pipe + 2 * KP;   // y buffer k drained
    cudaEvent_t ev_start = p->ev_pipe[3 * KP], ev_end = p->ev_pipe[3 * KP + 1];
    // the copy streams start after whatever the caller queued on `stream`
    if ((e = cudaEventRecord(ev_start, st))) return cuda_status(e, "event");
    cudaStreamWaitEvent(p->s_h2d, ev_start, 0);
    cudaStreamWaitEvent(p->s_d2h, ev_start, 0);
    spmv_status s = SPMV_OK;
    for (int32_t b = 0; b < count && !s; ++b) {
        const int k = b % NP;
        float* dx = p->d_hxb + k * (nx + ny);
        float* dy = dx + nx;
        if (b >= NP) cudaStreamWaitEvent(p->s_h2d, comp_done[k], 0);  // product b-NP done with dx
        if ((e = cudaMemcpyAsync(dx, xh + (int64_t)b * p->n_cols, p->n_cols * 4, cudaMemcpyHostToDevice, p->s_h2d)))
            { s = cuda_status(e, "H2D"); break; }
        cudaEventRecord(h2d_done[k], p->s_h2d);
        cudaStreamWaitEvent(st, h2d_done[k], 0);
        if (b >= NP) cudaStreamWaitEvent(st, d2h_done[k], 0);           // y of product b-NP drained
        if ((s = spmv_execute(p, dx, dy, stream))) break;
        cudaEventRecord(comp_done[k], st);
        cudaStreamWaitEvent(p->s_d2h, comp_done[k], 0);
        if ((e = cudaMemcpyAsync(yh + (int64_t)b * p->n_rows, dy, p->n_rows * 4, cudaMemcpyDeviceToHost, p->s_d2h)))
            { s = cuda_status(e, "D2H"); break; }
        cudaEventRecord(d2h_done[k], p->s_d2h);
    }
    // `stream` completes only after the last copy out
    cudaEventRecord(ev_end, p->s_d2h);
    cudaStreamWaitEvent(st, ev_end, 0);
    if ((e = cudaStreamSynchronize(st)) && !s) s = cuda_status(e, "sync");
    return s;
}

__attribute__((visibility("default")))
spmv_status spmv_execute_timed(spmv_plan p, const float* x, float* y, void* stream,
                               float* launch_ms, int32_t max_launches) {
    if (!p || !x || !y || !launch_ms) { set_error("null argument"); return SPMV_EINVAL; }
    if (p->device < 0) { set_error("host-only plan cannot execute"); return SPMV_EINVAL; }
    cudaError_t e = cudaSetDevice(p->device);
    if (e) return cuda_status(e, "cudaSetDevice");
    cudaStream_t st = (cudaStream_t)stream;
    if ((e = scratch_acquire(p, st))) return cuda_status(e, "scratch order");
    std::vector<cudaEvent_t> ev;
    auto mark = [&]() { cudaEvent_t v; cudaEventCreate(&v); cudaEventRecord(v, st); ev.push_back(v); };
    mark();
    if (p->two_phase) {
        const float* xa = pb_x(p, x, st, e);
        if (!e) e = launch_pb(*p, p->pb_grid, xa, EpiStore{y}, st);
        mark();
    } else if (p->n_cols > 0) {
        launch_permute(p, x, st);
        mark();
    }
    for (int32_t t = 0; t <= p->num_tiles && !p->two_phase; ++t) {
        if (p->tiles[t].wl_end == p->tiles[t].wl_begin) continue;
        if ((e = launch_tile(*p, t, p->grid_tile[t], p->d_xp, EpiStore{y}, st))) break;
        mark();
    }
    if (!e) e = scratch_release(p, st);
    if (!e) e = cudaStreamSynchronize(st);
    for (size_t i = 1; i < ev.size(); ++i) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ev[i - 1], ev[i]);
        if ((int32_t)(i - 1) < max_launches) launch_ms[i - 1] = ms;
    }
    for (auto v : ev) cudaEventDestroy(v);
    return cuda_status(e, "spmv_execute_timed");
}

__attribute__((visibility("default")))
spmv_status spmv_pb_trace(spmv_plan p, const float* x, float* y, void* stream, int64_t* trace_host,
                          int64_t n_items) {
    if (!p || !x || !y || !trace_host) { set_error("null argument"); return SPMV_EINVAL; }
    if (!p->two_phase || p->device < 0) { set_error("not a device two-phase plan"); return SPMV_EINVAL; }
    const int64_t ni = (int64_t)p->PB.items.size();
    if (n_items < ni) { set_error("trace buffer too small"); return SPMV_EINVAL; }
    cudaError_t e = cudaSetDevice(p->device);
    if (e) return cuda_status(e, "cudaSetDevice");
    cudaStream_t st = (cudaStream_t)stream;
    int64_t* d = nullptr;
    if ((e = cudaMalloc(&d, std::max<int64_t>(ni, 1) * 4 * sizeof(int64_t)))) return cuda_status(e, "trace");
    cudaMemsetAsync(d, 0, std::max<int64_t>(ni, 1) * 4 * sizeof(int64_t), st);
    const float* xa = pb_x(p, x, st, e);
    if (e || (e = scratch_acquire(p, st)) || (e = launch_pb(*p, p->pb_grid, xa, EpiStore{y}, st, d)) ||
        (e = scratch_release(p, st)) || (e = cudaStreamSynchronize(st)) ||
        (e = cudaMemcpy(trace_host, d, ni * 4 * sizeof(int64_t), cudaMemcpyDeviceToHost))) {
        cudaFree(d); return cuda_status(e, "trace run");
    }
    cudaFree(d);
    return SPMV_OK;
}

__attribute__((visibility("default")))
int32_t spmv_plan_launches(spmv_plan p) {
    if (!p) return 0;
    if (p->two_phase) return 1;
    int32_t n = p->n_cols > 0 ? 1 : 0;
    for (auto& t : p->tiles) n += (t.wl_end > t.wl_begin) ? 1 : 0;
    return n;
}

__attribute__((visibility("default")))
spmv_status spmv_plan_stats(spmv_plan p, spmv_plan_stats_t* o) {
    if (!p || !o) { set_error("null argument"); return SPMV_EINVAL; }
    std::memset(o, 0, sizeof(*o));
    o->n_rows = p->n_rows; o->n_cols = p->n_cols; o->nnz = p->nnz;
    o->num_tiles = p->num_tiles; o->tile_width = p->tile_width;
    o->n_workloads = p->n_workloads; o->n_slots = p->n_slots; o->n_row_entries = p->n_row_entries;
    o->n_split = p->n_split; o->n_chunks = p->n_chunks; o->device_bytes = p->device_bytes;
    o->predicted_us = p->predicted_us; o->build_ms = p->build_ms;
    for (int32_t t = 0; t <= p->num_tiles && t < 64; ++t) {
        const TileInfo& ti = p->tiles[t];
        o->wl[t] = ti.wl; o->tile_nnz[t] = ti.nnz; o->tile_rows[t] = ti.rows;
        o->tile_col_lo[t] = ti.col_lo; o->tile_col_hi[t] = ti.col_hi; o->tile_staged[t] = ti.staged;
        o->tile_predicted_us[t] = ti.pred_us; o->composite_threshold[t] = ti.threshold;
    }
    o->resident_warps = p->grid_tile.empty() ? 0 : p->grid_tile.back() * kWarps;
    o->perf_table_loaded = p->perf_table_loaded;
    o->two_phase = p->two_phase ? 1 : 0;
    o->orient = p->orient;
    o->pb_groups = p->pb_groups; o->pb_chunks = p->pb_chunks; o->pb_bins = p->pb_bins; o->pb_long_bins = p->pb_long;
    o->one_pass_predicted_us = p->one_pass_us; o->two_phase_predicted_us = p->two_phase_us;
    if (p->two_phase) o->resident_warps = p->pb_grid * kPbWarps;
    return SPMV_OK;
}

__attribute__((visibility("default")))
spmv_status spmv_plan_layout(spmv_plan p, spmv_layout_view* v) {
    if (!p || !v) { set_error("null argument"); return SPMV_EINVAL; }
    if (p->two_phase) { set_error("two-phase plan: no one-pass tile layout (use spmv_plan_to_coo)"); return SPMV_EINVAL; }
    spmv_status s = ensure_host(p);
    if (s) return s;
    HostLayout& L = p->L;
    const int64_t nw = p->n_workloads;
    L.v_tiles.resize(4 * (p->num_tiles + 1));
    for (int32_t t = 0; t <= p->num_tiles; ++t) {
        L.v_tiles[4 * t] = p->tiles[t].col_lo; L.v_tiles[4 * t + 1] = p->tiles[t].col_hi;
        L.v_tiles[4 * t + 2] = p->tiles[t].wl_begin; L.v_tiles[4 * t + 3] = p->tiles[t].wl_end;
    }
    L.v_off.resize(nw); L.v_row_base.resize(nw); L.v_w.resize(nw); L.v_h.resize(nw);
    L.v_split_id.resize(nw); L.v_chunk.resize(nw); L.v_kind.resize(nw); L.v_kvec.resize(nw);
    for (int64_t j = 0; j < nw; ++j) {
        const WlDesc& d = L.desc[j];
        L.v_off[j] = d.off; L.v_row_base[j] = d.row_base; L.v_w[j] = d.w; L.v_h[j] = d.h;
        L.v_split_id[j] = d.split_id; L.v_chunk[j] = d.chunk; L.v_kind[j] = d.kind; L.v_kvec[j] = d.kvec;
    }
    v->n_cols = p->n_cols; v->n_workloads = nw; v->n_row_entries = p->n_row_entries;
    v->n_slots = p->n_slots; v->n_split = p->n_split; v->n_tiles_total = p->num_tiles + 1;
    v->perm = p->perm.data(); v->tiles = L.v_tiles.data();
    v->desc_off = L.v_off.data(); v->desc_row_base = L.v_row_base.data(); v->desc_w = L.v_w.data();
    v->desc_h = L.v_h.data(); v->desc_split_id = L.v_split_id.data(); v->desc_chunk = L.v_chunk.data();
    v->desc_kind = L.v_kind.data(); v->desc_kvec = L.v_kvec.data();
    v->row_id = L.row_id.data(); v->slot_col = L.slot_col.data();
    v->slot_val = p->pattern ? nullptr : L.slot_val.data();
    v->split = L.split.data();
    return SPMV_OK;
}

__attribute__((visibility("default")))
spmv_status spmv_plan_export(spmv_plan p, const char* path) {
    if (!p || !path) { set_error("null argument"); return SPMV_EINVAL; }
    spmv_layout_view v;
    spmv_status s = spmv_plan_layout(p, &v);
    if (s) return s;
    FILE* f = std::fopen(path, "wb");
    if (!f) { set_error(std::string("cannot open ") + path); return SPMV_ENOMEM; }
    bool ok = true;
    auto put = [&](const void* a, size_t bytes) { if (bytes && ok) ok = std::fwrite(a, 1, bytes, f) == bytes; };
    const char magic[8] = {'T', 'C', 'S', 'P', 'M', 'V', '1', 0};
    const int64_t hdr[8] = {p->n_rows, v.n_cols, v.n_workloads, v.n_row_entries, v.n_slots, v.n_split,
                            v.n_tiles_total, p->pattern ? 0 : 1};
    const size_t nw = (size_t)v.n_workloads;
    put(magic, 8); put(hdr, sizeof(hdr));
    put(v.perm, 4 * (size_t)v.n_cols); put(v.tiles, 32 * (size_t)v.n_tiles_total);
    put(v.desc_off, 8 * nw); put(v.desc_row_base, 4 * nw); put(v.desc_w, 4 * nw); put(v.desc_h, 4 * nw);
    put(v.desc_split_id, 4 * nw); put(v.desc_chunk, 4 * nw); put(v.desc_kind, nw); put(v.desc_kvec, nw);
    put(v.row_id, 4 * (size_t)v.n_row_entries); put(v.slot_col, 4 * (size_t)v.n_slots);
    if (!p->pattern) put(v.slot_val, 4 * (size_t)v.n_slots);
    put(v.split, 12 * (size_t)v.n_split);
    if (std::fclose(f) != 0) ok = false;
    if (!ok) { set_error(std::string("short write to ") + path); return SPMV_ENOMEM; }
    return SPMV_OK;
}

// Read a Format v1 file written by spmv_plan_export and upload it (plan checkpoint / resume,
// the sort and packing are preprocessing, paid once per matrix).
__attribute__((visibility("default")))
spmv_status spmv_plan_import(const char* path, int device, spmv_plan* out) {
    if (!path || !out) { set_error("null argument"); return SPMV_EINVAL; }
    *out = nullptr;
    FILE* f = std::fopen(path, "rb");
    if (!f) { set_error(std::string("cannot open ") + path); return SPMV_EINVAL; }
    bool ok = true;
    auto get = [&](void* a, size_t bytes) { if (bytes && ok) ok = std::fread(a, 1, bytes, f) == bytes; };
    char magic[8] = {0};
    int64_t hdr[8] = {0};
    get(magic, 8); get(hdr, sizeof(hdr));
    if (!ok || std::memcmp(magic, "TCSPMV1", 8) != 0) { std::fclose(f); set_error("not a Format v1 plan file"); return SPMV_EINVAL; }
    const int64_t n_rows = hdr[0], n_cols = hdr[1], nw = hdr[2], ne = hdr[3], ns = hdr[4], nsp = hdr[5], nt = hdr[6];
    const bool valued = hdr[7] != 0;
    if (n_rows < 0 || n_cols < 0 || nw < 0 || ne < 0 || ns < 0 || nsp < 0 || nt < 1 || nt > 64) {
        std::fclose(f); set_error("plan file header out of range"); return SPMV_EINVAL;
    }
    spmv_plan_s* p = nullptr;
    try {
        p = new spmv_plan_s();
        p->n_rows = n_rows; p->n_cols = n_cols; p->pattern = !valued; p->device = device;
        spmv_options_default(&p->opt);
        p->opt.pattern = p->pattern ? 1 : 0;
        p->perm.resize(n_cols); get(p->perm.data(), 4 * (size_t)n_cols);
        std::vector<int64_t> tiles(4 * nt); get(tiles.data(), 32 * (size_t)nt);
        std::vector<int64_t> off(nw); std::vector<int32_t> rb(nw), w(nw), h(nw), sid(nw), ch(nw);
        std::vector<uint8_t> kind(nw), kvec(nw);
        get(off.data(), 8 * nw); get(rb.data(), 4 * nw); get(w.data(), 4 * nw); get(h.data(), 4 * nw);
        get(sid.data(), 4 * nw); get(ch.data(), 4 * nw); get(kind.data(), nw); get(kvec.data(), nw);
        HostLayout& L = p->L;
        L.row_id.resize(ne); get(L.row_id.data(), 4 * (size_t)ne);
        L.slot_col.resize(ns); get(L.slot_col.data(), 4 * (size_t)ns);
        if (valued) { L.slot_val.resize(ns); get(L.slot_val.data(), 4 * (size_t)ns); }
        L.split.resize(3 * nsp); get(L.split.data(), 12 * (size_t)nsp);
        std::fclose(f); f = nullptr;
        if (!ok) { delete p; set_error("short plan file"); return SPMV_EINVAL; }
        L.desc.resize(nw);
        for (int64_t j = 0; j < nw; ++j) {
            WlDesc& d = L.desc[j];
            d.off = off[j]; d.row_base = rb[j]; d.w = w[j]; d.h = h[j]; d.kind = kind[j]; d.kvec = kvec[j];
            d.pad_ = 0; d.split_id = sid[j]; d.chunk = ch[j];
        }
        p->num_tiles = (int32_t)(nt - 1);
        p->tiles.resize(nt);
        int64_t nnz = 0;
        for (int64_t t = 0; t < nt; ++t) {
            TileInfo& ti = p->tiles[t];
            ti.col_lo = tiles[4 * t]; ti.col_hi = tiles[4 * t + 1]; ti.wl_begin = tiles[4 * t + 2]; ti.wl_end = tiles[4 * t + 3];
            const int32_t sent = (int32_t)(ti.col_hi - ti.col_lo);
            for (int64_t j = ti.wl_begin; j < ti.wl_end; ++j) {
                const WlDesc& d = L.desc[j];
                const int64_t span = (int64_t)d.w * d.h;
                for (int64_t k = 0; k < span; ++k) ti.nnz += L.slot_col[d.off + k] != sent;
            }
            nnz += ti.nnz;
            if (t < nt - 1)
                ti.staged = (ti.col_hi - ti.col_lo) * 4 <= 227 * 1024 && ti.col_lo % 4 == 0;
        }
        p->tile_width = nt > 1 ? (int32_t)(p->tiles[0].col_hi - p->tiles[0].col_lo) : (int32_t)std::min<int64_t>(n_cols, INT32_MAX);
        p->nnz = nnz;
        p->n_workloads = nw; p->n_slots = ns; p->n_row_entries = ne; p->n_split = nsp;
        int64_t nch = 0;
        for (int64_t i = 0; i < nsp; ++i) nch = std::max<int64_t>(nch, (int64_t)L.split[3 * i + 2] + L.split[3 * i + 1]);
        p->n_chunks = L.n_chunks = nch;
        p->host_valid = true;
        if (device >= 0) {
            int ndev = 0;
            cudaError_t e = cudaGetDeviceCount(&ndev);
            if (e != cudaSuccess || ndev == 0) { delete p; set_error("no CUDA device"); return SPMV_ECUDA; }
            if (device >= ndev) { delete p; set_error("device ordinal out of range"); return SPMV_EINVAL; }
            if ((e = cudaSetDevice(device))) { delete p; return cuda_status(e, "cudaSetDevice"); }
            cudaDeviceGetAttribute(&p->sm_count, cudaDevAttrMultiProcessorCount, device);
            spmv_status st = upload_one_pass(p);
            if (st) return st;
        }
    } catch (const std::bad_alloc&) {
        if (f) std::fclose(f);
        delete p;
        set_error("host allocation failed"); return SPMV_ENOMEM;
    }
    *out = p;
    return SPMV_OK;
}

__attribute__((visibility("default")))
spmv_status spmv_plan_to_coo(spmv_plan p, int32_t* rows, int32_t* cols, float* vals) {
    if (!p || (p->nnz > 0 && (!rows || !cols))) { set_error("null argument"); return SPMV_EINVAL; }
    if (p->two_phase) return pb_to_coo(p, rows, cols, vals);
    spmv_status s = ensure_host(p);
    if (s) return s;
    const HostLayout& L = p->L;
    const int64_t eh = p->opt.ell_h;
    int64_t w = 0;
    for (int32_t t = 0; t <= p->num_tiles; ++t) {
        const TileInfo& ti = p->tiles[t];
        const int32_t sent = (int32_t)(ti.col_hi - ti.col_lo);
        for (int64_t j = ti.wl_begin; j < ti.wl_end; ++j) {
            const WlDesc& d = L.desc[j];
            auto put = [&](uint32_t ent, int64_t slot) {
                int32_t c = (int32_t)((uint32_t)L.slot_col[slot] & ~COO_END);
                if (c == sent) return;
                if (w >= p->nnz) return;
                rows[w] = (int32_t)(ent & ROW_MASK);
                cols[w] = p->perm[ti.col_lo + c];
                if (vals) vals[w] = p->pattern ? 1.0f : L.slot_val[slot];
                ++w;
            };
            if (d.kind == KIND_COO) {           // rows back to back, COO_END closes each
                int32_t r = 0;
                for (int32_t k = 0; k < d.w && r < d.h; ++k) {
                    const int64_t slot = d.off + k;
                    put(L.row_id[d.row_base + r], slot);
                    if ((uint32_t)L.slot_col[slot] & COO_END) ++r;
                }
            } else if (d.kind != KIND_CM) {
                for (int32_t r = 0; r < d.h; ++r)
                    for (int32_t k = 0; k < d.w; ++k) put(L.row_id[d.row_base + r], d.off + (int64_t)r * d.w + k);
            } else {
                for (int32_t r = 0; r < d.h; ++r) {
                    uint32_t ent = L.row_id[d.row_base + r];
                    if (ent == PAD_ROW) continue;
                    int64_t s0 = d.off + (int64_t)(r / eh) * eh * d.w, rr = r % eh;
                    for (int32_t k = 0; k < d.w; ++k)
                        put(ent, s0 + (k / d.kvec) * eh * d.kvec + rr * d.kvec + (k % d.kvec));
                }
            }
        }
    }
    if (w != p->nnz) { set_error("layout decode count mismatch"); return SPMV_EINVAL; }
    return SPMV_OK;
}

__attribute__((visibility("default"))) const char* spmv_last_error(void) { return g_last_error.c_str(); }
__attribute__((visibility("default"))) const char* spmv_version(void) { return "tcspmv 0.1 (sm_100a)"; }

}  // extern "C"
