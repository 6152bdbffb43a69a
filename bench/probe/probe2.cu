// Hardware probe 2: random gathers from distributed shared memory (thread-block clusters) vs
// local shared memory vs L2, on B200.  Not part of the product path.
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

constexpr int LOCAL = 49152;   // floats per CTA

// indices are global within the cluster segment [0, C*LOCAL)
__global__ void dsmem_gather(const int4* __restrict__ idx, int64_t rows, int K4, const float* __restrict__ x,
                             float* __restrict__ y, int csize) {
    extern __shared__ float xs[];
    cg::cluster_group cl = cg::this_cluster();
    unsigned rank = cl.block_rank();
    for (int i = threadIdx.x; i < LOCAL; i += blockDim.x) xs[i] = x[rank * LOCAL + i];
    cl.sync();
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += stride) {
        float acc = 0.f;
        for (int k = 0; k < K4; ++k) {
            int4 c = __ldcs(idx + (int64_t)k * rows + r);
            int cc[4] = {c.x, c.y, c.z, c.w};
            #pragma unroll
            for (int j = 0; j < 4; ++j) {
                unsigned owner = (unsigned)cc[j] / LOCAL, off = (unsigned)cc[j] % LOCAL;
                float* p = cl.map_shared_rank(xs, owner);
                acc += p[off];
            }
        }
        y[r] = acc;
    }
    cl.sync();
}

static uint64_t sm64(uint64_t z) { z += 0x9E3779B97F4A7C15ull; z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull; z = (z ^ (z >> 27)) * 0x94D049BB133111EBull; return z ^ (z >> 31); }

int main() {
    cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
    const int64_t rows = 1 << 22; const int K4 = 4;
    int64_t nidx = rows * K4 * 4;
    std::vector<int> hidx(nidx);
    float* dx; CK(cudaMalloc(&dx, 16 * LOCAL * 4)); CK(cudaMemset(dx, 0, 16 * LOCAL * 4));
    float* dy; CK(cudaMalloc(&dy, rows * 4));
    int4* didx; CK(cudaMalloc(&didx, nidx * 4));
    CK(cudaFuncSetAttribute(dsmem_gather, cudaFuncAttributeMaxDynamicSharedMemorySize, LOCAL * 4));
    CK(cudaFuncSetAttribute(dsmem_gather, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    int csizes[] = {1, 2, 4, 8, 16};
    for (int ci = 0; ci < 5; ++ci) {
        int C = csizes[ci];
        for (int64_t i = 0; i < nidx; ++i) hidx[i] = (int)(sm64(i * 31 + C) % (uint64_t)(C * LOCAL));
        CK(cudaMemcpy(didx, hidx.data(), nidx * 4, cudaMemcpyHostToDevice));
        for (int bs : {512, 1024}) {
            cudaLaunchConfig_t cfg = {};
            int nclusters = 148 / C;
            cfg.gridDim = dim3(nclusters * C); cfg.blockDim = dim3(bs); cfg.dynamicSmemBytes = LOCAL * 4;
            cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
            cfg.attrs = at; cfg.numAttrs = 1;
            int ncl = 0;
            cudaError_t oe = cudaOccupancyMaxActiveClusters(&ncl, dsmem_gather, &cfg);
            if (oe != cudaSuccess) { printf("{\"C\":%d,\"bs\":%d,\"occ_err\":\"%s\"}\n", C, bs, cudaGetErrorString(oe)); cudaGetLastError(); continue; }
            cfg.gridDim = dim3(ncl * C);
            float best = 1e9;
            for (int rep = 0; rep < 4; ++rep) {
                CK(cudaEventRecord(e0));
                cudaError_t le = cudaLaunchKernelEx(&cfg, dsmem_gather, (const int4*)didx, rows, K4, (const float*)dx, dy, C);
                if (le != cudaSuccess) { printf("launch err %s\n", cudaGetErrorString(le)); break; }
                CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
                float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); if (rep && ms < best) best = ms;
            }
            CK(cudaGetLastError());
            printf("{\"probe\":\"dsmem_gather\",\"C\":%d,\"bs\":%d,\"clusters\":%d,\"ms\":%.3f,\"Ggather_s\":%.1f}\n",
                   C, bs, ncl, best, nidx / best / 1e6);
        }
    }
    return 0;
}
