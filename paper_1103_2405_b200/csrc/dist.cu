// dist.cu -- multi-GPU row partitioning (Sec. 3.2): bitonic partition and
// the NCCL communicator (NCCL is loaded at run time with dlopen, so the library has no link-time
// dependency on a particular libnccl).
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <string>
#include <thread>
#include <cstring>
#include <memory>
#include <mutex>
#include <numeric>
#include <vector>

#include "epilogues.cuh"
#include "graph_build.h"
#include "launch.cuh"
#include "solver.h"
#include "trace.h"

using namespace tc;

// ------------------------------------------------------------------ NCCL (runtime loaded)
namespace {
typedef struct { char internal[128]; } NcclUid;
typedef void* NcclComm;
enum { ncclFloat32 = 7, ncclFloat64 = 8, ncclSum = 0 };
struct Nccl {
    void* h = nullptr;
    int (*GetUniqueId)(NcclUid*) = nullptr;
    int (*CommInitRank)(NcclComm*, int, NcclUid, int) = nullptr;
    int (*CommDestroy)(NcclComm) = nullptr;
    int (*AllGather)(const void*, void*, size_t, int, NcclComm, cudaStream_t) = nullptr;
    int (*AllReduce)(const void*, void*, size_t, int, int, NcclComm, cudaStream_t) = nullptr;
    int (*Send)(const void*, size_t, int, int, NcclComm, cudaStream_t) = nullptr;
    int (*Recv)(void*, size_t, int, int, NcclComm, cudaStream_t) = nullptr;
    int (*GroupStart)() = nullptr;
    int (*GroupEnd)() = nullptr;
    int (*CommGetAsyncError)(NcclComm, int*) = nullptr;
    int (*CommAbort)(NcclComm) = nullptr;
    const char* (*GetErrorString)(int) = nullptr;
    bool load() {
        if (h) return true;
        const char* names[] = {"libnccl.so.2", "libnccl.so"};
        for (const char* nm : names) {
            h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
            if (h) break;
        }
        if (!h) return false;
        GetUniqueId = (decltype(GetUniqueId))dlsym(h, "ncclGetUniqueId");
        CommInitRank = (decltype(CommInitRank))dlsym(h, "ncclCommInitRank");
        CommDestroy = (decltype(CommDestroy))dlsym(h, "ncclCommDestroy");
        AllGather = (decltype(AllGather))dlsym(h, "ncclAllGather");
        AllReduce = (decltype(AllReduce))dlsym(h, "ncclAllReduce");
        GetErrorString = (decltype(GetErrorString))dlsym(h, "ncclGetErrorString");
        Send = (decltype(Send))dlsym(h, "ncclSend");
        Recv = (decltype(Recv))dlsym(h, "ncclRecv");
        GroupStart = (decltype(GroupStart))dlsym(h, "ncclGroupStart");
        GroupEnd = (decltype(GroupEnd))dlsym(h, "ncclGroupEnd");
        CommGetAsyncError = (decltype(CommGetAsyncError))dlsym(h, "ncclCommGetAsyncError");
        CommAbort = (decltype(CommAbort))dlsym(h, "ncclCommAbort");
        return GetUniqueId && CommInitRank && CommDestroy && AllGather && AllReduce && Send && Recv &&
               GroupStart && GroupEnd;
    }
};
Nccl g_nccl;
}  // namespace

// Loopback transport (test transport, spmv_comm_create_loopback): `world` logical ranks in one
// process on one device, one host thread and stream each.  The same exchange() interface moves the
// data with device-to-device copies: every rank publishes (buffer, event) at a host barrier, then
// pulls the pieces it receives from its peers' buffers on its own stream, and a second barrier
// (with the copies' events) keeps a peer from overwriting its slot before everyone has read it.
namespace {
struct Loopback {
    int world = 1;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    long gen = 0;
    std::vector<const void*> ptr;           // published buffer per rank
    std::vector<const int64_t*> offs;       // published per-peer offsets (needed mode)
    std::vector<cudaEvent_t> ready, done;   // per rank: data ready / copies out of it finished
    std::vector<std::vector<char>> host;    // metadata allgather
    // the ranks' solver builds run one at a time: they share one host, and a c5 slice build holds
    // several GB of host vectors (per-rank processes on a real box build on their own hosts' cores
    // in parallel; here the builder's OpenMP loops already use every core)
    std::mutex build_mu;
    // slices mode (spmv_comm_create_slices): the ranks are row slices of one solver on one device
    // and share one double-buffered exchange buffer -- each writes its own slot, and the exchange
    // is only the ordering (every rank waits for every other rank's slot), no copies
    bool shared = false;
    int device = 0;
    float* sG[2] = {nullptr, nullptr};      // mailbox: rank 0's solver posts its buffers at its first run
    int64_t sG_floats = -1;
    void barrier() {
        std::unique_lock<std::mutex> lk(mu);
        const long g = gen;
        if (++arrived == world) { arrived = 0; ++gen; cv.notify_all(); }
        else cv.wait(lk, [&] { return gen != g; });
    }
};
}  // namespace

struct spmv_comm_s {
    int rank = 0, world = 1, device = 0;
    NcclComm comm = nullptr;
    std::shared_ptr<Loopback> lb;           // loopback transport (no NCCL)
};

static spmv_status nccl_status(int r, const char* what) {
    if (r == 0) return SPMV_OK;
    set_error(std::string(what) + ": " + (g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "nccl error"));
    return SPMV_ENCCL;
}

// ids [0, n) ordered by (length desc, id asc): a stable counting sort over the lengths (O(n + max
// length); the c5 block has 267 M rows, where a comparison sort costs a minute per call)
template <class Len>
static std::vector<int64_t> order_by_length_desc(int64_t n, Len len) {
    int64_t mx = 0;
    for (int64_t i = 0; i < n; ++i) mx = std::max<int64_t>(mx, len(i));
    std::vector<int64_t> start(mx + 2, 0);
    for (int64_t i = 0; i < n; ++i) start[mx - len(i) + 1]++;        // bucket b = mx - length
    for (int64_t b = 0; b <= mx; ++b) start[b + 1] += start[b];
    std::vector<int64_t> order(n);
    for (int64_t i = 0; i < n; ++i) order[start[mx - len(i)]++] = i;
    return order;
}

extern "C" {

__attribute__((visibility("default")))
spmv_status bitonic_partition(int64_t n_rows, const int64_t* row_len, int32_t P, int32_t* owner) {
    if (n_rows < 0 || (n_rows > 0 && (!row_len || !owner)) || P < 1) { set_error("invalid argument"); return SPMV_EINVAL; }
    if (P > std::max<int64_t>(n_rows, 1)) { set_error("P > rows"); return SPMV_ERANGE; }
    // rows by (length desc, id asc); sorted position s -> s mod P on even rounds, P-1-(s mod P)
    // on odd rounds (the previous round's longest-row recipient gets the shortest row, L108)
    for (int64_t i = 0; i < n_rows; ++i)
        if (row_len[i] < 0) { set_error("negative row length"); return SPMV_EINVAL; }
    const std::vector<int64_t> order = order_by_length_desc(n_rows, [&](int64_t i) { return row_len[i]; });
    for (int64_t s = 0; s < n_rows; ++s) {
        int64_t g = s / P, j = s % P;
        owner[order[s]] = (int32_t)((g % 2 == 0) ? j : P - 1 - j);
    }
    return SPMV_OK;
}

// Row ownership and slot layout of the row-partitioned path (Sec. 3.2): owner by bitonic
// partition; inside a rank its rows keep ascending id order (local_index); every rank's slot
// holds slot_rows entries (the largest rank count, so the allgather has equal counts).
__attribute__((visibility("default")))
spmv_status spmv_partition_plan(int64_t n_rows, const int64_t* row_len, int32_t P, int32_t* owner,
                                int64_t* local_index, int64_t* slot_rows) {
    spmv_status s = bitonic_partition(n_rows, row_len, P, owner);
    if (s) return s;
    if (!local_index || !slot_rows) { set_error("null argument"); return SPMV_EINVAL; }
    std::vector<int64_t> cnt(P, 0);
    for (int64_t i = 0; i < n_rows; ++i) local_index[i] = cnt[owner[i]]++;
    *slot_rows = n_rows ? *std::max_element(cnt.begin(), cnt.end()) : 0;
    return SPMV_OK;
}

// Needed-columns exchange lists: rank r sends to q the values of the vertices r
// owns that q's rows read; it receives from q the values of q's vertices its own rows read.
// Both lists ascending by vertex id, so sender and receiver agree on the order without talking.
static void needed_lists_impl(int64_t n, const int64_t* rp, const int32_t* col, const int32_t* owner,
                              int32_t P, int32_t rank, std::vector<std::vector<int32_t>>& send,
                              std::vector<std::vector<int32_t>>& recv) {
    send.assign(P, {});
    recv.assign(P, {});
    std::vector<int32_t> stamp(n, -1);
    // rows grouped by owner (ascending id within a rank)
    std::vector<int64_t> cnt(P + 1, 0);
    for (int64_t i = 0; i < n; ++i) cnt[owner[i] + 1]++;
    for (int32_t q = 0; q < P; ++q) cnt[q + 1] += cnt[q];
    std::vector<int64_t> rows(n), fill(cnt.begin(), cnt.end() - 1);
    for (int64_t i = 0; i < n; ++i) rows[fill[owner[i]]++] = i;
    for (int32_t q = 0; q < P; ++q) {
        if (q == rank) continue;
        std::vector<int32_t>& out = send[q];
        for (int64_t t = cnt[q]; t < cnt[q + 1]; ++t) {
            const int64_t i = rows[t];
            for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
                const int32_t v = col[k];
                if (owner[v] == rank && stamp[v] != q) { stamp[v] = q; out.push_back(v); }
            }
        }
        std::sort(out.begin(), out.end());
    }
    std::fill(stamp.begin(), stamp.end(), -1);
    for (int64_t t = cnt[rank]; t < cnt[rank + 1]; ++t) {
        const int64_t i = rows[t];
        for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
            const int32_t v = col[k];
            if (owner[v] != rank && stamp[v] != rank) { stamp[v] = rank; recv[owner[v]].push_back(v); }
        }
    }
    for (auto& r : recv) std::sort(r.begin(), r.end());
}

__attribute__((visibility("default")))
spmv_status spmv_needed_lists(int64_t n, const int64_t* row_ptr, const int32_t* col, const int32_t* owner,
                              int32_t P, int32_t rank, int64_t* send_count, int64_t* recv_count,
                              int32_t* send_ids, int32_t* recv_ids) {
    if (n < 0 || (n > 0 && (!row_ptr || !owner)) || P < 1 || rank < 0 || rank >= P || !send_count || !recv_count) {
        set_error("invalid argument"); return SPMV_EINVAL;
    }
    for (int64_t i = 0; i < n; ++i)
        if (owner[i] < 0 || owner[i] >= P) { set_error("owner out of range"); return SPMV_ERANGE; }
    if (n > 0 && row_ptr[n] > 0 && !col) { set_error("null col"); return SPMV_EINVAL; }
    for (int64_t k = 0; k < (n > 0 ? row_ptr[n] : 0); ++k)
        if (col[k] < 0 || col[k] >= n) { set_error("column out of range"); return SPMV_EINVAL; }
    try {
        std::vector<std::vector<int32_t>> send, recv;
        needed_lists_impl(n, row_ptr, col, owner, P, rank, send, recv);
        int64_t so = 0, ro = 0;
        for (int32_t q = 0; q < P; ++q) {
            send_count[q] = (int64_t)send[q].size();
            recv_count[q] = (int64_t)recv[q].size();
            if (send_ids) std::copy(send[q].begin(), send[q].end(), send_ids + so);
            if (recv_ids) std::copy(recv[q].begin(), recv[q].end(), recv_ids + ro);
            so += send_count[q]; ro += recv_count[q];
        }
    } catch (const std::bad_alloc&) { set_error("host allocation failed"); return SPMV_ENOMEM; }
    return SPMV_OK;
}

__attribute__((visibility("default"))) spmv_status spmv_comm_unique_id(void* id_out) {
    if (!id_out) { set_error("null argument"); return SPMV_EINVAL; }
    if (!g_nccl.load()) { set_error("libnccl.so.2 not found"); return SPMV_ENCCL; }
    NcclUid u;
    spmv_status s = nccl_status(g_nccl.GetUniqueId(&u), "ncclGetUniqueId");
    if (!s) std::memcpy(id_out, &u, sizeof(u));
    return s;
}

__attribute__((visibility("default")))
spmv_status spmv_comm_create(int rank, int world, const void* uid, int device, spmv_comm* out) {
    if (!out || world < 1 || rank < 0 || rank >= world || (world > 1 && !uid)) { set_error("invalid argument"); return SPMV_EINVAL; }
    cudaError_t e = cudaSetDevice(device);
    if (e) return cuda_status(e, "cudaSetDevice");
    spmv_comm_s* c = new spmv_comm_s();
    c->rank = rank; c->world = world; c->device = device;
    if (world > 1) {
        if (!g_nccl.load()) { delete c; set_error("libnccl.so.2 not found"); return SPMV_ENCCL; }
        NcclUid u;
        std::memcpy(&u, uid, sizeof(u));
        spmv_status s = nccl_status(g_nccl.CommInitRank(&c->comm, world, u, rank), "ncclCommInitRank");
        if (s) { delete c; return s; }
    }
    *out = c;
    return SPMV_OK;
}

static spmv_status create_loopback(int world, int device, bool shared, spmv_comm* out) {
    if (!out || world < 1) { set_error("invalid argument"); return SPMV_EINVAL; }
    cudaError_t e = cudaSetDevice(device);
    if (e) return cuda_status(e, "cudaSetDevice");
    auto lb = std::make_shared<Loopback>();
    lb->world = world;
    lb->shared = shared;
    lb->device = device;
    lb->ptr.assign(world, nullptr);
    lb->offs.assign(world, nullptr);
    lb->ready.assign(world, nullptr);
    lb->done.assign(world, nullptr);
    lb->host.assign(world, {});
    for (int r = 0; r < world; ++r) {
        if ((e = cudaEventCreateWithFlags(&lb->ready[r], cudaEventDisableTiming)) ||
            (e = cudaEventCreateWithFlags(&lb->done[r], cudaEventDisableTiming))) {
            for (auto ev : lb->ready) if (ev) cudaEventDestroy(ev);
            for (auto ev : lb->done) if (ev) cudaEventDestroy(ev);
            return cuda_status(e, "loopback events");
        }
    }
    for (int r = 0; r < world; ++r) {
        spmv_comm_s* c = new spmv_comm_s();
        c->rank = r; c->world = world; c->device = device; c->lb = lb;
        out[r] = c;
    }
    return SPMV_OK;
}

__attribute__((visibility("default")))
spmv_status spmv_comm_create_loopback(int world, int device, spmv_comm* out) {
    return create_loopback(world, device, false, out);
}

__attribute__((visibility("default")))
spmv_status spmv_comm_create_slices(int world, int device, spmv_comm* out) {
    return create_loopback(world, device, true, out);
}

__attribute__((visibility("default"))) void spmv_comm_destroy(spmv_comm c) {
    if (!c) return;
    if (c->comm) g_nccl.CommDestroy(c->comm);
    if (c->lb && c->lb.use_count() == 1) {
        for (auto ev : c->lb->ready) if (ev) cudaEventDestroy(ev);
        for (auto ev : c->lb->done) if (ev) cudaEventDestroy(ev);
    }
    delete c;
}

}  // extern "C"


// ------------------------------------------------------------------ row-partitioned solvers
namespace {

struct Dist {
    int P = 1, rank = 0;
    uint8_t* d_half_local = nullptr;         // HITS: half flag per local row
    uint8_t* d_col_half = nullptr;           // HITS: per G position 0 / 1 = half of its vertex, 2 = no value
    int64_t n_local = 0, S = 0, slot = 0;    // owned rows, exchanged rows per slot, slot floats (S + partials)
    int64_t S_full = 0;                      // owned rows per slot of the one-time result gather
    int64_t g_floats = 0;                    // exchange buffer length (the local plan's x)
    std::vector<int64_t> gpos;               // vertex -> position in the gathered buffer (-1: never exchanged)
    std::vector<int64_t> gpos_full;          // vertex -> position in the result gather
    std::vector<int32_t> owned;              // local row -> vertex
    std::vector<int64_t> lrow;               // vertex -> local row index on its owner
    int64_t q_local = -1;
    // exchange buffer, double buffered: iteration k reads x from d_Gb[k & 1] (the local plan's
    // columns are G positions) while its epilogue writes the next x into d_Gb[(k + 1) & 1]'s own
    // slot; P slots (needed mode: own slot + P-1 segments)
    float* d_Gb[2] = {nullptr, nullptr};
    int64_t* d_part_off = nullptr;           // [P] offset of rank q's fp64 partials in d_G
    // needed-columns exchange (spmv_iter_opts.exchange = 1)
    int exchange = 0;
    std::vector<int64_t> soff, scnt, roff, rcnt;   // per peer: send / receive segment (floats, incl. partials)
    float* d_S = nullptr;                    // send buffer
    int32_t* d_sidx = nullptr;               // send position -> own slot position (-1: padding)
    int64_t n_send = 0;
    bool shared = false;                     // slices mode: d_Gb shared by every rank's solver
    bool owns_shared = false;                //   allocated (and freed) by rank 0's solver
};

// send buffer: S[i] = own slot[sidx[i]] (values of the vertices a peer reads, then the partials)
__global__ void dist_pack(const float* __restrict__ slot, const int32_t* __restrict__ sidx, float* __restrict__ S,
                          int64_t n, const tc::Ctrl* ctrl) {
    if (*(volatile const int32_t*)&ctrl->done) return;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t j = __ldg(sidx + i);
        S[i] = j >= 0 ? slot[j] : 0.0f;
    }
}

constexpr int64_t kPartialFloats = 8;        // four fp64 partials, 16-byte multiple

// sum the P ranks' partials in rank order (identical on every rank: deterministic), advance
__global__ void dist_finalize(const float* G, const int64_t* part_off, int P, tc::Ctrl* ctrl, int rwr) {
    if (threadIdx.x != 0 || *(volatile int32_t*)&ctrl->done) return;
    double res = 0.0, dm = 0.0;
    for (int r = 0; r < P; ++r) {
        const double* part = reinterpret_cast<const double*>(G + part_off[r]);
        res += part[0];
        dm += part[1];
    }
    if (!rwr) ctrl->tele = ctrl->c * dm * ctrl->inv_n + (1.0 - ctrl->c) * ctrl->inv_n;
    ctrl->dmass = dm;
    ctrl->residual = res;
    ctrl->iter += 1;
    bool done = ctrl->fixed_iters > 0 ? ctrl->iter >= ctrl->fixed_iters : (res < ctrl->tol || ctrl->iter >= ctrl->max_iter);
    ctrl->done = done ? 1 : 0;
}

__global__ void dist_init(float* p, float* zslot, const float* inv, int64_t n_local, int rwr,
                          int64_t q_local, float p0) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_local; i += (int64_t)gridDim.x * blockDim.x) {
        float v = rwr ? (i == q_local ? 1.0f : 0.0f) : p0;
        p[i] = v;
        if (inv[i] != 0.0f) zslot[i] = v * inv[i];   // empty columns (inv = 0) are not exchanged
    }
}

// slot[r] = p_e[fpos[r]]: the local rows' values out of row-entry order
__global__ void gather_rows(const float* p_e, const int32_t* fpos, float* slot, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        slot[i] = fpos[i] >= 0 ? p_e[fpos[i]] : 0.0f;
}

// HITS (Eq. 8) row-partitioned: the slots carry the raw product y and the half sums; every rank
// derives the same half norms (rank-order sums), normalises its own rows (post) and the gathered
// x it reads (permute).  The L1 change of a normalisation travels with the next exchange, so the
// stop decision lags one SpMV and the reported iterate is the one that converged (reading R14).
__global__ void hits_dist_finalize(const float* G, const int64_t* part_off, int P, tc::Ctrl* ctrl, int l2) {
    if (threadIdx.x != 0 || *(volatile int32_t*)&ctrl->done) return;
    double s0 = 0.0, s1 = 0.0, r = 0.0;
    for (int k = 0; k < P; ++k) {
        const double* part = reinterpret_cast<const double*>(G + part_off[k]);
        s0 += part[0]; s1 += part[1]; r += part[2];
    }
    if (ctrl->iter >= 1) {
        ctrl->residual = r;
        const bool done = ctrl->fixed_iters > 0 ? ctrl->iter >= ctrl->fixed_iters
                                                : (r < ctrl->tol || ctrl->iter >= ctrl->max_iter);
        if (done) { ctrl->done = 1; return; }
    }
    ctrl->norm[0] = l2 ? sqrt(s0) : s0;
    ctrl->norm[1] = l2 ? sqrt(s1) : s1;
    ctrl->iter += 1;
}

// own rows: v = y / |y_half| (zero half -> uniform, R5); L1 change into the own slot's partial 2
__global__ void __launch_bounds__(512) hits_dist_post(float* slot_y, float* v_old, const uint8_t* half, int64_t n_local,
                                                      tc::Ctrl* ctrl, double* slots, double* res_out) {
    if (*(volatile int32_t*)&ctrl->done) return;
    const double n0 = ctrl->norm[0], n1 = ctrl->norm[1];
    const float uni = (float)ctrl->uniform;
    const float s0 = n0 > 0.0 ? (float)(1.0 / n0) : 0.0f, s1 = n1 > 0.0 ? (float)(1.0 / n1) : 0.0f;
    double res = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_local; i += (int64_t)gridDim.x * blockDim.x) {
        const int h = half[i];
        const double nn = h ? n1 : n0;
        const float vn = nn > 0.0 ? slot_y[i] * (h ? s1 : s0) : uni;
        res += fabs((double)vn - (double)v_old[i]);
        v_old[i] = vn;
    }
    double acc[1] = {res};
    tc::block_reduce_to_slot<1>(acc, slots + blockIdx.x);
    if (!tc::last_block(&ctrl->ticket)) return;
    double s[1];
    tc::block_sum_slots<1>(slots, gridDim.x, s);
    if (threadIdx.x == 0) { ctrl->ticket = 0; *res_out = s[0]; }
}

// the gathered raw products normalised in place (they are the next x, read by the SpMV straight
// from G): v = y / |y_half|, a zero half -> uniform (R5); partial and padding positions kept
__global__ void hits_dist_scale(float* __restrict__ G, const uint8_t* __restrict__ gh, int64_t n,
                                const tc::Ctrl* ctrl) {
    if (*(volatile const int32_t*)&ctrl->done) return;
    const double n0 = ctrl->norm[0], n1 = ctrl->norm[1];
    const float uni = (float)ctrl->uniform;
    const float s0 = n0 > 0.0 ? (float)(1.0 / n0) : 0.0f, s1 = n1 > 0.0 ? (float)(1.0 / n1) : 0.0f;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        const int h = gh[k];
        if (h == 2) continue;
        const double nn = h ? n1 : n0;
        G[k] = nn > 0.0 ? G[k] * (h ? s1 : s0) : uni;
    }
}

// every value position of G set to v (HITS a(0) = h(0) = 1/|V|, L440)
__global__ void g_fill_values(float* __restrict__ G, const uint8_t* __restrict__ gh, int64_t n, float v) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
        if (gh[k] != 2) G[k] = v;
}

__global__ void fill_f(float* a, int64_t n, float v) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) a[i] = v;
}

// loopback: pull piece q of every peer q into `dst` (src_q + soff(q) -> dst + doff(q), n(q) floats)
template <class Src, class Dst, class Cnt>
spmv_status loopback_pull(spmv_comm c, const void* mine, const int64_t* my_offs, Src src_off, Dst dst_off, Cnt cnt,
                          float* dst, cudaStream_t st) {
    Loopback& L = *c->lb;
    const int r = c->rank;
    cudaError_t e = cudaEventRecord(L.ready[r], st);
    L.ptr[r] = mine;
    L.offs[r] = my_offs;
    L.barrier();                                        // every peer's data is enqueued
    for (int q = 0; q < c->world && !e; ++q) {
        if (q == r || cnt(q) == 0) continue;
        if (!(e = cudaStreamWaitEvent(st, L.ready[q], 0)))
            e = cudaMemcpyAsync(dst + dst_off(q), static_cast<const float*>(L.ptr[q]) + src_off(q, L.offs[q]),
                                (size_t)cnt(q) * sizeof(float), cudaMemcpyDeviceToDevice, st);
    }
    if (!e) e = cudaEventRecord(L.done[r], st);
    L.barrier();                                        // every copy out of our buffer is enqueued
    for (int q = 0; q < c->world && !e; ++q)
        if (q != r) e = cudaStreamWaitEvent(st, L.done[q], 0);
    L.barrier();                                        // events free for the next round
    return cuda_status(e, "loopback exchange");
}

// Failure detection: wait for the stream while polling NCCL's asynchronous error
// state; a peer failure or a hang past the watchdog aborts the communicator (the collective
// kernels would otherwise spin forever) and returns SPMV_ENCCL instead of blocking.
constexpr double kWatchdogSeconds = 600.0;
spmv_status wait_stream(spmv_comm c, cudaStream_t st, const char* what) {
    const auto t0 = std::chrono::steady_clock::now();
    for (;;) {
        const cudaError_t q = cudaStreamQuery(st);
        if (q == cudaSuccess) return SPMV_OK;
        if (q != cudaErrorNotReady) return cuda_status(q, what);
        if (c && c->comm) {
            int ae = 0;
            if (g_nccl.CommGetAsyncError && g_nccl.CommGetAsyncError(c->comm, &ae) == 0 && ae != 0) {
                if (g_nccl.CommAbort) g_nccl.CommAbort(c->comm);
                c->comm = nullptr;
                return nccl_status(ae, "NCCL asynchronous error (communicator aborted)");
            }
        }
        const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (el > kWatchdogSeconds) {
            if (c && c->comm && g_nccl.CommAbort) { g_nccl.CommAbort(c->comm); c->comm = nullptr; }
            set_error(std::string(what) + ": watchdog (" + std::to_string((int)kWatchdogSeconds) + " s) expired");
            return c && c->world > 1 ? SPMV_ENCCL : SPMV_ECUDA;
        }
        std::this_thread::sleep_for(std::chrono::microseconds(100));
    }
}

spmv_status allgather(spmv_comm c, float* G, int64_t slot, cudaStream_t st) {
    if (c->world == 1) return SPMV_OK;
    if (c->lb)
        return loopback_pull(c, G, nullptr, [&](int q, const int64_t*) { return (int64_t)q * slot; },
                             [&](int q) { return (int64_t)q * slot; }, [&](int) { return slot; }, G, st);
    return nccl_status(g_nccl.AllGather(G + (int64_t)c->rank * slot, G, (size_t)slot, ncclFloat32, c->comm, st),
                       "ncclAllGather");
}

// slices mode: every rank's stream waits for every other rank's work enqueued so far (its slot of
// the shared buffer written); two host barriers around the waits, as in loopback_pull
spmv_status sync_ranks(spmv_comm c, cudaStream_t st) {
    Loopback& L = *c->lb;
    const int r = c->rank;
    cudaError_t e = cudaEventRecord(L.ready[r], st);
    L.barrier();
    for (int q = 0; q < c->world && !e; ++q)
        if (q != r) e = cudaStreamWaitEvent(st, L.ready[q], 0);
    L.barrier();                                        // events free for the next round
    return cuda_status(e, "slices sync");
}

// the per-iteration exchange: one in-place allgather of equal slots, or (needed mode) the packed
// per-peer segments by grouped point-to-point sends / receives; slices mode: ordering only
spmv_status exchange(spmv_comm c, Dist* D, float* G, const tc::Ctrl* ctrl, int sm_count, cudaStream_t st) {
    tc::Range r("exchange");
    if (D->shared) return c->world == 1 ? SPMV_OK : sync_ranks(c, st);
    if (!D->exchange) return allgather(c, G, D->slot, st);
    if (c->world == 1) return SPMV_OK;
    if (D->n_send) dist_pack<<<sm_count * 2, 256, 0, st>>>(G, D->d_sidx, D->d_S, D->n_send, ctrl);
    if (c->lb) {
        // rank q's segment for us sits at q's soff[rank]; it lands at our roff[q]
        const int me = D->rank;
        return loopback_pull(c, D->d_S, D->soff.data(), [&](int, const int64_t* offs) { return offs[me]; },
                             [&](int q) { return D->roff[q]; }, [&](int q) { return D->rcnt[q]; }, G, st);
    }
    spmv_status s = nccl_status(g_nccl.GroupStart(), "ncclGroupStart");
    for (int q = 0; q < D->P && !s; ++q) {
        if (q == D->rank) continue;
        s = nccl_status(g_nccl.Send(D->d_S + D->soff[q], (size_t)D->scnt[q], ncclFloat32, q, c->comm, st), "ncclSend");
        if (!s) s = nccl_status(g_nccl.Recv(G + D->roff[q], (size_t)D->rcnt[q], ncclFloat32, q, c->comm, st), "ncclRecv");
    }
    spmv_status e = nccl_status(g_nccl.GroupEnd(), "ncclGroupEnd");
    return s ? s : e;
}

}  // namespace


// metadata allgather of the local-input variant (host vectors through device buffers, NCCL)
static spmv_status allgather_host(spmv_comm c, const void* mine, void* all, size_t count, int dtype, size_t esize) {
    if (c->world == 1) { std::memcpy(all, mine, count * esize); return SPMV_OK; }
    if (c->lb) {
        Loopback& L = *c->lb;
        L.host[c->rank].assign((const char*)mine, (const char*)mine + count * esize);
        L.barrier();
        for (int q = 0; q < c->world; ++q) std::memcpy((char*)all + (size_t)q * count * esize, L.host[q].data(), count * esize);
        L.barrier();
        return SPMV_OK;
    }
    void* d = nullptr;
    cudaError_t e = cudaMalloc(&d, count * esize * c->world);
    if (e) return cuda_status(e, "metadata buffer");
    spmv_status s = SPMV_OK;
    e = cudaMemcpy((char*)d + (size_t)c->rank * count * esize, mine, count * esize, cudaMemcpyHostToDevice);
    if (e) s = cuda_status(e, "metadata upload");
    if (!s) s = nccl_status(g_nccl.AllGather((char*)d + (size_t)c->rank * count * esize, d, count, dtype, c->comm, nullptr),
                            "ncclAllGather (metadata)");
    if (!s && (e = cudaDeviceSynchronize())) s = cuda_status(e, "metadata allgather");
    if (!s && (e = cudaMemcpy(all, d, count * esize * c->world, cudaMemcpyDeviceToHost))) s = cuda_status(e, "metadata download");
    cudaFree(d);
    return s;
}

spmv_status solver_create_dist(int algo, int64_t n, int64_t m, const int64_t* row_ptr,
                               const int32_t* col, const spmv_iter_opts* it,
                               const spmv_options* opt_in, spmv_comm comm, int device,
                               spmv_solver* out, const LocalInput* li) {
    (void)m;
    cudaError_t e = cudaSetDevice(device);
    if (e) return cuda_status(e, "cudaSetDevice");
    spmv_solver_s* s = new spmv_solver_s();
    Dist* D = new Dist();
    s->algo = algo; s->n = n; s->N = n; s->device = device; s->comm = comm; s->dist = D;
    if (it) s->it = *it; else spmv_iter_opts_default(&s->it, algo);
    D->P = comm->world; D->rank = comm->rank;
    spmv_status st = SPMV_OK;
    std::unique_lock<std::mutex> build_lock;       // loopback: one rank's build at a time
    try {
        std::vector<int64_t> mrp, len; std::vector<int32_t> mcol;
        std::vector<int32_t> owner;
        std::vector<int64_t> rl;                  // full input: row length of every vertex
        std::vector<int64_t> in_row;              // local input: vertex -> input row (-1: not ours)
        int64_t S = 0;
        const int64_t nv = n;
        if (!li) {
            if (comm->lb) build_lock = std::unique_lock<std::mutex>(comm->lb->build_mu);
            std::vector<int64_t> arp; std::vector<int32_t> acol;
            clean_adjacency(n, row_ptr, col, arp, acol);
            n = build_iteration_matrix(algo, nv, arp, acol, mrp, mcol, len);   // n := vector length N
            // partition rows of M (bitonic over row lengths, Sec. 3.2)
            rl.resize(n);
            for (int64_t i = 0; i < n; ++i) rl[i] = mrp[i + 1] - mrp[i];
            owner.resize(n);
            std::vector<int64_t> lidx(n);
            if ((st = spmv_partition_plan(n, rl.data(), D->P, owner.data(), lidx.data(), &S))) throw st;
        } else {
            // local input (SURVEY 8(b) "*_local"): this rank's rows only; ownership and the
            // degrees of every vertex come from one metadata allgather (O(n) per rank, not O(m))
            const int64_t nl = li->n_local;
            std::vector<int64_t> counts(D->P);
            if ((st = allgather_host(comm, &nl, counts.data(), 1, 4 /*ncclInt64*/, 8))) throw st;
            const int64_t mx = *std::max_element(counts.begin(), counts.end());
            S = mx;
            std::vector<int32_t> mine(2 * std::max<int64_t>(mx, 1), -1), all(2 * std::max<int64_t>(mx, 1) * D->P);
            for (int64_t r = 0; r < nl; ++r) {
                mine[r] = li->owned[r];
                mine[mx + r] = li->out_degree ? li->out_degree[r]
                                              : (int32_t)(li->row_ptr[r + 1] - li->row_ptr[r]);
            }
            if ((st = allgather_host(comm, mine.data(), all.data(), 2 * std::max<int64_t>(mx, 1), 2 /*ncclInt32*/, 4))) throw st;
            std::vector<int32_t>().swap(mine);
            if (comm->lb) build_lock = std::unique_lock<std::mutex>(comm->lb->build_mu);
            // HITS: the rows are those of the block matrix [[0, A^T], [A, 0]] (Eq. 8),
            // 2|V| of them; a row's length is also its column's length (the block is structurally
            // symmetric), so it orders the exchange slots like the full-input path's column lengths
            if (algo == SPMV_ALGO_HITS) n = 2 * nv;
            owner.assign(n, -1);
            len.assign(n, 0);
            const int64_t w = 2 * std::max<int64_t>(mx, 1);
            for (int32_t q = 0; q < D->P; ++q)
                for (int64_t r = 0; r < counts[q]; ++r) {
                    const int32_t v = all[q * w + r];
                    if (v < 0 || v >= n || owner[v] != -1) { set_error("owned ids overlap or out of range"); throw SPMV_EINVAL; }
                    owner[v] = q;
                    len[v] = all[q * w + mx + r];
                }
            std::vector<int32_t>().swap(all);
            for (int64_t v = 0; v < n; ++v)
                if (owner[v] < 0) { set_error("a vertex is owned by no rank"); throw SPMV_EINVAL; }
            in_row.assign(n, -1);
            for (int64_t r = 0; r < nl; ++r) in_row[li->owned[r]] = r;
        }
        s->N = n;
        auto row_len = [&](int64_t v) -> int64_t {
            return li ? li->row_ptr[in_row[v] + 1] - li->row_ptr[in_row[v]] : rl[v];
        };
        auto row_cols = [&](int64_t v) -> const int32_t* {
            return li ? li->col + li->row_ptr[in_row[v]] : mcol.data() + mrp[v];
        };
        // Exchange only globally non-empty columns: for PageRank / RWR a column of
        // the iteration matrix is empty exactly when the vertex has no out-edges (inv = 0), so its
        // z is never read.  On each rank the non-empty rows come first (ascending id), then the
        // rest; the exchanged slot holds the first part only.  HITS exchanges every row.
        std::vector<char> col_ne(n, algo == SPMV_ALGO_HITS ? 1 : 0);
        if (algo != SPMV_ALGO_HITS)
            for (int64_t u = 0; u < n; ++u) col_ne[u] = len[u] != 0;
        std::vector<int64_t> cnt_ne(D->P, 0), cnt_all(D->P, 0);
        for (int64_t i = 0; i < n; ++i) { cnt_ne[owner[i]] += col_ne[i]; cnt_all[owner[i]]++; }
        // Rank-contiguous relabel: rank q's vertices occupy slot q of the exchange buffer G, ordered
        // by (column length desc, id asc) -- the non-empty columns first, the densest first
        // (Solution 2, L66, inside each slot).  The local plan reads G itself as its x (columns
        // given in G positions, keep_col_order), so no per-iteration gather builds x from G.
        D->lrow.resize(n);
        {
            const std::vector<int64_t> order = order_by_length_desc(n, [&](int64_t i) { return len[i]; });
            std::vector<int64_t> next(D->P, 0);
            for (int64_t i : order) D->lrow[i] = next[owner[i]]++;
        }
        const int64_t S_ex = n ? *std::max_element(cnt_ne.begin(), cnt_ne.end()) : 0;
        D->S = (S_ex + 3) / 4 * 4;
        D->slot = D->S + kPartialFloats;
        D->S_full = std::max<int64_t>(S, 1);
        D->gpos.resize(n);
        D->gpos_full.resize(n);
        D->owned.assign(cnt_all[D->rank], 0);
        #pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; ++i) {
            D->gpos[i] = col_ne[i] ? (int64_t)owner[i] * D->slot + D->lrow[i] : -1;
            D->gpos_full[i] = (int64_t)owner[i] * D->S_full + D->lrow[i];
            if (owner[i] == D->rank) D->owned[D->lrow[i]] = (int32_t)i;
        }
        D->n_local = (int64_t)D->owned.size();
        // exchange layout: allgather slots, or (needed columns) the own slot then
        // one segment per peer holding the values of its vertices our rows read (ascending id,
        // padded to 4 floats) + its partials
        std::vector<int64_t> part_off(D->P);
        int64_t g_floats = (int64_t)D->P * D->slot;
        D->exchange = s->it.exchange == 1;
        if (D->exchange && li) { set_error("exchange = 1 needs the full graph on every rank"); throw SPMV_EINVAL; }
        D->shared = comm->lb && comm->lb->shared;
        if (D->exchange && D->shared) { set_error("slices share one exchange buffer: exchange = 0 only"); throw SPMV_EINVAL; }
        std::vector<std::vector<int32_t>> recv;
        if (!D->exchange) {
            for (int32_t q = 0; q < D->P; ++q) part_off[q] = (int64_t)q * D->slot + D->S;
        } else {
            std::vector<std::vector<int32_t>> send;
            needed_lists_impl(n, mrp.data(), mcol.data(), owner.data(), D->P, D->rank, send, recv);
            D->soff.assign(D->P, 0); D->scnt.assign(D->P, 0); D->roff.assign(D->P, 0); D->rcnt.assign(D->P, 0);
            int64_t ro = D->slot, so = 0;
            std::vector<int32_t> sidx;
            for (int32_t q = 0; q < D->P; ++q) {
                if (q == D->rank) { part_off[q] = D->S; continue; }
                const int64_t rp4 = ((int64_t)recv[q].size() + 3) / 4 * 4;
                D->roff[q] = ro; D->rcnt[q] = rp4 + kPartialFloats; part_off[q] = ro + rp4; ro += D->rcnt[q];
                const int64_t sp4 = ((int64_t)send[q].size() + 3) / 4 * 4;
                D->soff[q] = so; D->scnt[q] = sp4 + kPartialFloats; so += D->scnt[q];
                for (int32_t v : send[q]) sidx.push_back((int32_t)D->lrow[v]);
                for (int64_t j = (int64_t)send[q].size(); j < sp4; ++j) sidx.push_back(-1);
                for (int64_t j = 0; j < kPartialFloats; ++j) sidx.push_back((int32_t)(D->S + j));
            }
            g_floats = ro;
            D->n_send = so;
            if (so) {
                if ((e = cudaMalloc(&D->d_S, so * sizeof(float))) || (e = cudaMalloc(&D->d_sidx, so * sizeof(int32_t))) ||
                    (e = cudaMemcpy(D->d_sidx, sidx.data(), so * sizeof(int32_t), cudaMemcpyHostToDevice))) {
                    st = cuda_status(e, "needed-columns buffers"); throw st;
                }
            }
        }
        D->g_floats = g_floats;
        // G position of the value of vertex v that this rank's rows read
        auto gcol = [&](int64_t v) -> int64_t {
            if (!D->exchange) return D->gpos[v];
            const int32_t q = owner[v];
            if (q == D->rank) return D->lrow[v];
            auto it = std::lower_bound(recv[q].begin(), recv[q].end(), (int32_t)v);
            if (it == recv[q].end() || *it != v) return -1;
            return D->roff[q] + (it - recv[q].begin());
        };
        // local rows (lrow order), columns as G positions
        std::vector<int64_t> lrp(D->n_local + 1, 0);
        for (int64_t r = 0; r < D->n_local; ++r) lrp[r + 1] = lrp[r] + row_len(D->owned[r]);
        std::vector<int32_t> lcol(lrp[D->n_local]);
        {
            // one pass over this rank's entries (c5: 1.4 G per rank), threads over rows
            int bad = 0;
            #pragma omp parallel for schedule(dynamic, 4096) reduction(|:bad)
            for (int64_t r = 0; r < D->n_local; ++r) {
                const int64_t v = D->owned[r];
                const int32_t* c = row_cols(v);
                const int64_t L = row_len(v);
                for (int64_t k = 0; k < L; ++k) {
                    if (c[k] < 0 || c[k] >= n) { bad |= 1; break; }
                    const int64_t gp = gcol(c[k]);
                    if (gp < 0) { bad |= 2; break; }
                    lcol[lrp[r] + k] = (int32_t)gp;
                }
            }
            if (bad & 1) { set_error("column out of range"); throw SPMV_EINVAL; }
            if (bad & 2) { set_error("internal: referenced column not exchanged"); throw SPMV_EINVAL; }
        }
        spmv_options opt;
        if (opt_in) opt = *opt_in; else spmv_options_default(&opt);
        opt.pattern = 1;
        opt.two_phase = 0;         // the row-partitioned epilogue runs on the one-pass tiles
        opt.keep_col_order = 1;    // x is G itself
        opt.num_tiles = -1; opt.tile_width = 0;
        if ((st = tc::create_plan(D->n_local, g_floats, lrp[D->n_local], lrp.data(), lcol.data(), nullptr, &opt, device, &s->plan))) throw st;
        spmv_plan_s* p = s->plan;
        std::vector<float> inv(std::max<int64_t>(D->n_local, 1), 0.0f);
        int64_t n_dangling = 0;
        for (int64_t u = 0; u < n; ++u) n_dangling += (len[u] == 0);
        for (int64_t r = 0; r < D->n_local; ++r) {
            const int64_t v = D->owned[r];
            inv[r] = len[v] ? (float)(1.0 / (double)len[v]) : 0.0f;
        }
        s->n_dangling = n_dangling;
#define CKD(x) do { if ((e = (x)) != cudaSuccess) { st = cuda_status(e, #x); throw st; } } while (0)
        for (int b = 0; b < 2 && !D->shared; ++b) {     // slices: shared buffers, set up at the first run
            CKD(cudaMalloc(&D->d_Gb[b], (size_t)g_floats * sizeof(float)));
            CKD(cudaMemset(D->d_Gb[b], 0, (size_t)g_floats * sizeof(float)));
        }
        CKD(cudaMalloc(&D->d_part_off, D->P * sizeof(int64_t)));
        CKD(cudaMemcpy(D->d_part_off, part_off.data(), D->P * sizeof(int64_t), cudaMemcpyHostToDevice));
        const int64_t nl = std::max<int64_t>(D->n_local, 1);
        CKD(cudaMalloc(&s->d_p, (nl + 4) * sizeof(float)));
        CKD(cudaMalloc(&s->d_y, (nl + 4) * sizeof(float)));
        CKD(cudaMalloc(&s->d_inv, nl * sizeof(float)));
        CKD(cudaMemcpy(s->d_inv, inv.data(), nl * sizeof(float), cudaMemcpyHostToDevice));
        CKD(cudaMalloc(&s->d_ctrl, sizeof(Ctrl)));
        CKD(cudaMemset(s->d_ctrl, 0, sizeof(Ctrl)));
        if (algo == SPMV_ALGO_HITS) {
            // per G position: 0 authority, 1 hub (vertex >= nv), 2 no value (partials, padding)
            std::vector<uint8_t> hl(nl, 0), ch(std::max<int64_t>(g_floats, 1), 2);
            for (int64_t r = 0; r < D->n_local; ++r) hl[r] = D->owned[r] >= nv;
            for (int64_t v = 0; v < n; ++v) {
                const int64_t gp = gcol(v);
                if (gp >= 0) ch[gp] = v >= nv;
            }
            CKD(cudaMalloc(&D->d_half_local, nl));
            CKD(cudaMemcpy(D->d_half_local, hl.data(), nl, cudaMemcpyHostToDevice));
            CKD(cudaMalloc(&D->d_col_half, ch.size()));
            CKD(cudaMemcpy(D->d_col_half, ch.data(), ch.size(), cudaMemcpyHostToDevice));
        }
        if (algo == SPMV_ALGO_HITS) CKD(setup_grids<EpiHitsSpmv>(*p, s->grids));
        else CKD(setup_grids<EpiAffine>(*p, s->grids));
        int32_t slots = 0;
        for (int32_t t = 0; t <= p->num_tiles; ++t) {
            if (p->tiles[t].wl_end == p->tiles[t].wl_begin) continue;
            s->tiles_used.push_back(t);
            s->slot_base.push_back(slots);
            slots += s->grids[t];
        }
        s->total_slots = slots;
        CKD(cudaMalloc(&s->d_slots, (size_t)std::max(slots, p->sm_count * 4) * 2 * sizeof(double)));
        std::vector<uint32_t> entries;
        if ((st = plan_final_positions(p, entries, s->fpos))) throw st;
        const int64_t ne = std::max<int64_t>(p->n_row_entries, 1);
        std::vector<float> inv_e(ne, 0.0f);
        std::vector<uint8_t> half_e(ne, 0);
        for (int64_t k = 0; k < p->n_row_entries; ++k) {
            const uint32_t ent = entries[k];
            if (ent != PAD_ROW && (ent & FLAG_FINAL)) {
                inv_e[k] = inv[ent & ROW_MASK];
                half_e[k] = D->owned[ent & ROW_MASK] >= nv;
            }
        }
        CKD(cudaMalloc(&s->d_half_e, ne));
        CKD(cudaMemcpy(s->d_half_e, half_e.data(), ne, cudaMemcpyHostToDevice));
        CKD(cudaMalloc(&s->d_p_e, ne * sizeof(float)));
        CKD(cudaMalloc(&s->d_inv_e, ne * sizeof(float)));
        CKD(cudaMemcpy(s->d_inv_e, inv_e.data(), ne * sizeof(float), cudaMemcpyHostToDevice));
        CKD(cudaMalloc(&s->d_fpos, nl * sizeof(int32_t)));
        if (D->n_local) CKD(cudaMemcpy(s->d_fpos, s->fpos.data(), D->n_local * sizeof(int32_t), cudaMemcpyHostToDevice));
        // per-vertex host tables the iteration does not read (c5: 2 GB each per rank)
        std::vector<int64_t>().swap(D->gpos);
        if (algo != SPMV_ALGO_RWR) std::vector<int64_t>().swap(D->lrow);
#undef CKD
    } catch (spmv_status code) {
        st = code;
    } catch (const std::bad_alloc&) {
        set_error("host allocation failed"); st = SPMV_ENOMEM;
    }
    if (st) { solver_destroy_dist(s); return st; }
    *out = s;
    return SPMV_OK;
}

spmv_status solver_run_dist(spmv_solver s, int64_t query, void* stream, spmv_iter_result* res) {
    tc::Range r_run("spmv_solver_run (row-partitioned)");
    Dist* D = static_cast<Dist*>(s->dist);
    spmv_plan_s* p = s->plan;
    if (s->algo == SPMV_ALGO_RWR && (query < 0 || query >= s->n)) { set_error("query out of range"); return SPMV_ERANGE; }
    cudaError_t e = cudaSetDevice(s->device);
    if (e) return cuda_status(e, "cudaSetDevice");
    cudaStream_t st = (cudaStream_t)stream;
    if (!st) {
        if (!s->own_stream && (e = cudaStreamCreateWithFlags(&s->own_stream, cudaStreamNonBlocking)))
            return cuda_status(e, "stream");
        st = s->own_stream;
    }
    const int rwr = s->algo == SPMV_ALGO_RWR;
    const int hitsa = s->algo == SPMV_ALGO_HITS;
    if (D->shared && !D->d_Gb[0]) {
        // slices mode, first run: rank 0 allocates the shared double buffer (owned by its solver)
        // and posts it; every rank picks it up between two barriers
        Loopback& L = *s->comm->lb;
        if (D->rank == 0) {
            float* b[2] = {nullptr, nullptr};
            const size_t bytes = (size_t)D->g_floats * sizeof(float);
            if (!cudaMalloc(&b[0], bytes) && !cudaMalloc(&b[1], bytes) && !cudaMemset(b[0], 0, bytes) &&
                !cudaMemset(b[1], 0, bytes) && !cudaDeviceSynchronize()) {
                L.sG[0] = b[0]; L.sG[1] = b[1]; L.sG_floats = D->g_floats;
                D->owns_shared = true;
            } else {
                cudaFree(b[0]); cudaFree(b[1]);
                L.sG[0] = L.sG[1] = nullptr; L.sG_floats = -1;
            }
        }
        L.barrier();
        const bool ok = L.sG[0] && L.sG_floats == D->g_floats;
        if (ok) { D->d_Gb[0] = L.sG[0]; D->d_Gb[1] = L.sG[1]; }
        L.barrier();                                   // the mailbox is free for the next solver
        if (!ok) { set_error("slices: shared exchange buffer unavailable"); return SPMV_ENOMEM; }
    }
    D->q_local = -1;
    if (rwr && D->lrow[query] < D->n_local && D->owned[D->lrow[query]] == (int32_t)query) D->q_local = D->lrow[query];
    Ctrl c{};
    const double n = (double)s->n;
    c.c = s->it.c; c.tol = s->it.tol; c.max_iter = s->it.max_iter; c.fixed_iters = s->it.fixed_iters;
    c.inv_n = 1.0 / n; c.residual = INFINITY; c.q = (int32_t)D->q_local;
    c.tele = rwr ? 0.0 : c.c * ((double)s->n_dangling / n) / n + (1.0 - c.c) / n;
    c.uniform = s->it.hits_norm == 1 ? 1.0 / n : 1.0 / std::sqrt(n);
    if ((e = cudaMemcpyAsync(s->d_ctrl, &c, sizeof(Ctrl), cudaMemcpyHostToDevice, st))) return cuda_status(e, "ctrl");
    // own slot of buffer b (where the epilogue writes the next x / raw product)
    auto own = [&](int b) { return D->exchange ? D->d_Gb[b] : D->d_Gb[b] + (int64_t)D->rank * D->slot; };
    const int g = p->sm_count * 4;
    spmv_status ss = SPMV_OK;
    // slices mode: a rank touches only its own slot of the shared buffer
    const int64_t own_lo = D->shared ? (int64_t)D->rank * D->slot : 0;
    const int64_t own_n = D->shared ? D->S : D->g_floats;
    if (hitsa) {   // a(0) = h(0) = 1/|V| (L440): own rows and every gathered column
        fill_f<<<g, 256, 0, st>>>(s->d_p, D->n_local, (float)(1.0 / n));
        g_fill_values<<<g, 256, 0, st>>>(D->d_Gb[0] + own_lo, D->d_col_half + own_lo, own_n, (float)(1.0 / n));
        if (D->shared && (ss = exchange(s->comm, D, D->d_Gb[0], s->d_ctrl, p->sm_count, st))) return ss;
    } else {
        dist_init<<<g, 256, 0, st>>>(s->d_p, own(0), s->d_inv, D->n_local, rwr, D->q_local, (float)(1.0 / n));
        init_entries<<<g, 256, 0, st>>>(s->d_p_e, p->d_row_id, p->n_row_entries, rwr, (int32_t)D->q_local, (float)(1.0 / n));
        if ((ss = exchange(s->comm, D, D->d_Gb[0], s->d_ctrl, p->sm_count, st))) return ss;
    }
    // host allocations before the first event: the GPU must not idle inside the timed region
    Ctrl* hc = nullptr;
    cudaMallocHost(&hc, sizeof(Ctrl));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0, st);
    const int batch = 8;
    const int cap = std::max(s->it.max_iter, s->it.fixed_iters) + batch;
    int launched = 0;
    // an event after every enqueued iteration: the reported time ends at the iteration that
    // converged, not at the batch's trailing (no-op kernels, but real exchanges) iterations
    std::vector<cudaEvent_t> ev_it;
    auto mark_iter = [&]() {
        cudaEvent_t v;
        cudaEventCreate(&v);
        cudaEventRecord(v, st);
        ev_it.push_back(v);
    };
    // phase boundaries of each iteration: after the local SpMV, after the exchange
    std::vector<cudaEvent_t> ev_spmv, ev_exch;
    auto mark = [&](std::vector<cudaEvent_t>& v) {
        cudaEvent_t x;
        cudaEventCreate(&x);
        cudaEventRecord(x, st);
        v.push_back(x);
    };
    while (true) {
        for (int b = 0; b < batch; ++b) {
            const size_t nu = s->tiles_used.size();
            float* Gx = D->d_Gb[launched & 1];          // this iteration's x
            float* Gn = D->d_Gb[(launched + 1) & 1];    // the next x (own slot written here, then exchanged)
            float* zslot = own((launched + 1) & 1);
            if (hitsa) {
                for (size_t i = 0; i < nu; ++i) {
                    EpiHitsSpmv epi{};
                    epi.y = zslot; epi.half = s->d_half_e; epi.fpos = s->d_fpos; epi.ctrl = s->d_ctrl;
                    epi.slots = s->d_slots; epi.slot_base = s->slot_base[i]; epi.total_slots = s->total_slots;
                    epi.is_last = (i + 1 == nu); epi.l2 = s->it.hits_norm != 1;
                    epi.dist_out = reinterpret_cast<double*>(zslot + D->S);
                    if ((e = launch_tile(*p, s->tiles_used[i], s->grids[s->tiles_used[i]], Gx, epi, st)))
                        return cuda_status(e, "tile launch");
                }
                if (nu == 0) cudaMemsetAsync(zslot + D->S, 0, 2 * sizeof(double), st);
                mark(ev_spmv);
                if ((ss = exchange(s->comm, D, Gn, s->d_ctrl, p->sm_count, st))) return ss;
                mark(ev_exch);
                hits_dist_finalize<<<1, 32, 0, st>>>(Gn, D->d_part_off, D->P, s->d_ctrl, s->it.hits_norm != 1);
                // the normalisation's L1 change travels with the NEXT exchange: it goes to the
                // partials of the buffer the next iteration writes its product into
                hits_dist_post<<<g, 512, 0, st>>>(zslot, s->d_p, D->d_half_local, D->n_local, s->d_ctrl, s->d_slots,
                                                  reinterpret_cast<double*>(own(launched & 1) + D->S) + 2);
                hits_dist_scale<<<g, 256, 0, st>>>(Gn + own_lo, D->d_col_half + own_lo, own_n, s->d_ctrl);
                // slices: the next SpMV reads every rank's normalised slot
                if (D->shared && (ss = exchange(s->comm, D, Gn, s->d_ctrl, p->sm_count, st))) return ss;
                mark_iter();
                ++launched;
                continue;
            }
            for (size_t i = 0; i < nu; ++i) {
                EpiAffine epi{};
                epi.y = s->d_y; epi.p = s->d_p_e; epi.z_next = zslot; epi.inv_deg = s->d_inv_e;
                epi.fpos = s->d_fpos;
                epi.ctrl = s->d_ctrl; epi.slots = s->d_slots; epi.slot_base = s->slot_base[i];
                epi.total_slots = s->total_slots; epi.is_last = (i + 1 == nu); epi.cond = 0;
                epi.rwr = rwr;
                epi.dist_out = reinterpret_cast<double*>(zslot + D->S);
                if ((e = launch_tile(*p, s->tiles_used[i], s->grids[s->tiles_used[i]], Gx, epi, st)))
                    return cuda_status(e, "tile launch");
            }
            if (nu == 0) cudaMemsetAsync(zslot + D->S, 0, 2 * sizeof(double), st);
            mark(ev_spmv);
            if ((ss = exchange(s->comm, D, Gn, s->d_ctrl, p->sm_count, st))) return ss;
            mark(ev_exch);
            dist_finalize<<<1, 32, 0, st>>>(Gn, D->d_part_off, D->P, s->d_ctrl, rwr);
            mark_iter();
            ++launched;
        }
        cudaMemcpyAsync(hc, s->d_ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, st);
        if ((ss = wait_stream(s->comm, st, "iteration loop"))) {
            cudaFreeHost(hc);
            for (auto v : ev_it) cudaEventDestroy(v);
            for (auto v : ev_spmv) cudaEventDestroy(v);
            for (auto v : ev_exch) cudaEventDestroy(v);
            return ss;
        }
        if (hc->done || launched > cap) break;
    }
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    c = *hc;
    // PageRank / RWR: iteration k ends with the k-th body; HITS decides to stop one body later
    // (the stop check lags one SpMV), so its converged run ends with body iter + 1
    int64_t last = hitsa ? (int64_t)c.iter : (int64_t)c.iter - 1;
    last = std::min<int64_t>(std::max<int64_t>(last, 0), (int64_t)ev_it.size() - 1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, last >= 0 ? ev_it[last] : e1);
    double ph[3] = {0.0, 0.0, 0.0};
    for (int64_t i = 0; i <= last; ++i) {
        float a = 0.f, b = 0.f, c3 = 0.f;
        cudaEventElapsedTime(&a, i ? ev_it[i - 1] : e0, ev_spmv[i]);
        cudaEventElapsedTime(&b, ev_spmv[i], ev_exch[i]);
        cudaEventElapsedTime(&c3, ev_exch[i], ev_it[i]);
        ph[0] += a; ph[1] += b; ph[2] += c3;
    }
    cudaEventDestroy(e0); cudaEventDestroy(e1);
    for (auto v : ev_it) cudaEventDestroy(v);
    for (auto v : ev_spmv) cudaEventDestroy(v);
    for (auto v : ev_exch) cudaEventDestroy(v);
    cudaFreeHost(hc);
    s->last = c;
    if (res) {
        res->iterations = c.iter; res->residual = c.residual;
        res->converged = s->it.fixed_iters > 0 ? 1 : (c.residual < s->it.tol);
        res->ms_total = ms; res->us_per_iter = c.iter ? 1000.0 * ms / c.iter : 0.0;
        res->predicted_us_per_iter = p->predicted_us;
        for (int k = 0; k < 3; ++k) res->phase_us[k] = last >= 0 ? 1000.0 * ph[k] / (double)(last + 1) : 0.0;
    }
    if (s->it.fixed_iters <= 0 && !(c.residual < s->it.tol)) { set_error("max_iter reached"); return SPMV_ENOCONV; }
    return SPMV_OK;
}

spmv_status solver_result_dist(spmv_solver s, float* out0, float* out1) {
    Dist* D = static_cast<Dist*>(s->dist);
    cudaSetDevice(s->device);
    cudaStream_t st = s->own_stream;
    // one-time gather of every owned row (the iteration exchange skips empty columns)
    float* d_R = nullptr;
    cudaError_t e = cudaMalloc(&d_R, (size_t)D->P * D->S_full * sizeof(float));
    if (e) return cuda_status(e, "result buffer");
    float* slot = d_R + (int64_t)D->rank * D->S_full;
    if (s->algo == SPMV_ALGO_HITS)
        cudaMemcpyAsync(slot, s->d_p, D->n_local * sizeof(float), cudaMemcpyDeviceToDevice, st);
    else
        gather_rows<<<s->plan->sm_count * 4, 256, 0, st>>>(s->d_p_e, s->d_fpos, slot, D->n_local);
    spmv_status ss = allgather(s->comm, d_R, D->S_full, st);
    if (ss) { cudaFree(d_R); return ss; }
    std::vector<float> G((size_t)D->P * D->S_full);
    e = cudaMemcpyAsync(G.data(), d_R, G.size() * sizeof(float), cudaMemcpyDeviceToHost, st);
    if (!e) e = cudaStreamSynchronize(st);
    cudaFree(d_R);
    if (e) return cuda_status(e, "result");
    for (int64_t u = 0; u < s->n; ++u) out0[u] = G[D->gpos_full[u]];
    if (s->algo == SPMV_ALGO_HITS)
        for (int64_t u = 0; u < s->n; ++u) out1[u] = G[D->gpos_full[s->n + u]];
    return SPMV_OK;
}

void solver_destroy_dist(spmv_solver s) {
    Dist* D = static_cast<Dist*>(s->dist);
    cudaSetDevice(s->device);
    if (D) {
        if (!D->shared || D->owns_shared) { cudaFree(D->d_Gb[0]); cudaFree(D->d_Gb[1]); }
        cudaFree(D->d_half_local); cudaFree(D->d_col_half);
        cudaFree(D->d_part_off); cudaFree(D->d_S); cudaFree(D->d_sidx);
        delete D;
    }
    if (s->own_stream) cudaStreamDestroy(s->own_stream);
    cudaFree(s->d_p); cudaFree(s->d_y); cudaFree(s->d_inv); cudaFree(s->d_ctrl); cudaFree(s->d_slots);
    cudaFree(s->d_p_e); cudaFree(s->d_inv_e); cudaFree(s->d_fpos);
    if (s->plan) spmv_plan_destroy(s->plan);
    delete s;
}
