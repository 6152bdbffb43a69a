// dist.cu -- multi-GPU row partitioning (Sec. 3.2): bitonic partition and
// the NCCL communicator (NCCL is loaded at run time with dlopen, so the library has no link-time
// dependency on a particular libnccl).
#include <dlfcn.h>

#include <algorithm>
#include <cstring>
#include <numeric>
#include <vector>

#include "solver.h"

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
        return GetUniqueId && CommInitRank && CommDestroy && AllGather && AllReduce;
    }
};
Nccl g_nccl;
}  // namespace

struct spmv_comm_s {
    int rank = 0, world = 1, device = 0;
    NcclComm comm = nullptr;
};

static spmv_status nccl_status(int r, const char* what) {
    if (r == 0) return SPMV_OK;
    set_error(std::string(what) + ": " + (g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "nccl error"));
    return SPMV_ENCCL;
}

extern "C" {

__attribute__((visibility("default")))
spmv_status bitonic_partition(int64_t n_rows, const int64_t* row_len, int32_t P, int32_t* owner) {
    if (n_rows < 0 || (n_rows > 0 && (!row_len || !owner)) || P < 1) { set_error("invalid argument"); return SPMV_EINVAL; }
    if (P > std::max<int64_t>(n_rows, 1)) { set_error("P > rows"); return SPMV_ERANGE; }
    // rows by (length desc, id asc); sorted position s -> s mod P on even rounds, P-1-(s mod P)
    // on odd rounds (the previous round's longest-row recipient gets the shortest row, L108)
    std::vector<int64_t> order(n_rows);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return row_len[a] > row_len[b]; });
    for (int64_t s = 0; s < n_rows; ++s) {
        int64_t g = s / P, j = s % P;
        owner[order[s]] = (int32_t)((g % 2 == 0) ? j : P - 1 - j);
    }
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

__attribute__((visibility("default"))) void spmv_comm_destroy(spmv_comm c) {
    if (!c) return;
    if (c->comm) g_nccl.CommDestroy(c->comm);
    delete c;
}

}  // extern "C"

spmv_status solver_create_dist(int, int64_t, int64_t, const int64_t*, const int32_t*,
                               const spmv_iter_opts*, const spmv_options*, spmv_comm, int,
                               spmv_solver*) {
    set_error("multi-GPU solver: not built in this version");
    return SPMV_EINVAL;
}
spmv_status solver_run_dist(spmv_solver, int64_t, void*, spmv_iter_result*) {
    set_error("multi-GPU solver: not built in this version");
    return SPMV_EINVAL;
}
spmv_status solver_result_dist(spmv_solver, float*, float*) {
    set_error("multi-GPU solver: not built in this version");
    return SPMV_EINVAL;
}
void solver_destroy_dist(spmv_solver) {}
