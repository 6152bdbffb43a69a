// Hardware probe: stream bandwidth and random-gather rates on B200.
// Not part of the product path.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__global__ void stream_read(const int4* __restrict__ a, int64_t n4, float* out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int acc = 0;
    for (; i < n4; i += stride) { int4 v = __ldcs(a + i); acc ^= v.x ^ v.y ^ v.z ^ v.w; }
    if (acc == 0x12345678) out[0] = 1.f;
}

template <int MODE>   // 0: ld.global (L1 alloc) 1: ld.global.nc.L1::no_allocate 2: smem-staged x
__global__ void ell_gather(const int4* __restrict__ idx, int64_t rows, int K4, const float* __restrict__ x,
                           int S, float* __restrict__ y) {
    extern __shared__ float xs[];
    if (MODE == 2) {
        for (int i = threadIdx.x; i < S; i += blockDim.x) xs[i] = x[i];
        __syncthreads();
    }
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += stride) {
        float acc = 0.f;
        for (int k = 0; k < K4; ++k) {
            int4 c = __ldcs(idx + (int64_t)k * rows + r);
            float v0, v1, v2, v3;
            if (MODE == 0) { v0 = x[c.x]; v1 = x[c.y]; v2 = x[c.z]; v3 = x[c.w]; }
            else if (MODE == 1) {
                asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v0) : "l"(x + c.x));
                asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v1) : "l"(x + c.y));
                asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v2) : "l"(x + c.z));
                asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v3) : "l"(x + c.w));
            } else { v0 = xs[c.x]; v1 = xs[c.y]; v2 = xs[c.z]; v3 = xs[c.w]; }
            acc += (v0 + v1) + (v2 + v3);
        }
        y[r] = acc;
    }
}

static uint64_t sm64(uint64_t z) { z += 0x9E3779B97F4A7C15ull; z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull; z = (z ^ (z >> 27)) * 0x94D049BB133111EBull; return z ^ (z >> 31); }

int main() {
    cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
    printf("{\"device\":\"%s\",\"sms\":%d,\"l2_bytes\":%d,\"persist_l2_max\":%d,\"smem_optin\":%zu,\"smem_per_sm\":%zu,\"max_thr_sm\":%d,\"clock_khz\":%d}\n",
           prop.name, prop.multiProcessorCount, prop.l2CacheSize, prop.persistingL2CacheMaxSize,
           prop.sharedMemPerBlockOptin, prop.sharedMemPerMultiprocessor, prop.maxThreadsPerMultiProcessor, prop.clockRate);
    cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
    float* dout; CK(cudaMalloc(&dout, 4));
    // stream
    int64_t nb = 2ll << 30; int4* buf; CK(cudaMalloc(&buf, nb)); CK(cudaMemset(buf, 1, nb));
    for (int rep = 0; rep < 3; ++rep) {
        CK(cudaEventRecord(e0)); stream_read<<<148 * 8, 256>>>(buf, nb / 16, dout); CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1)); float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
        if (rep == 2) printf("{\"probe\":\"stream_read\",\"GBps\":%.1f}\n", nb / ms / 1e6);
    }
    CK(cudaFree(buf));
    // gather
    const int64_t rows = 1 << 24; const int K4 = 4;   // 16 indices per row, 256M... (64M idx = 256 MB)
    int64_t nidx = rows * K4 * 4;
    std::vector<int> hidx(nidx);
    int sizes[] = {49152, 1 << 20, 4847571, 41291594};
    float* dx; CK(cudaMalloc(&dx, (size_t)41291594 * 4 + 64)); CK(cudaMemset(dx, 0, (size_t)41291594 * 4));
    float* dy; CK(cudaMalloc(&dy, rows * 4));
    int4* didx; CK(cudaMalloc(&didx, nidx * 4));
    CK(cudaFuncSetAttribute(ell_gather<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    for (int dist = 0; dist < 2; ++dist)
    for (int si = 0; si < 4; ++si) {
        int S = sizes[si];
        for (int64_t i = 0; i < nidx; ++i) {
            uint64_t r = sm64(i * 7919 + dist * 1000003 + S);
            double u = (r >> 11) * (1.0 / 9007199254740992.0);
            hidx[i] = dist == 0 ? (int)(u * S) : (int)(S * u * u * u * u);  // skew: hot low ids
            if (hidx[i] >= S) hidx[i] = S - 1;
        }
        CK(cudaMemcpy(didx, hidx.data(), nidx * 4, cudaMemcpyHostToDevice));
        for (int mode = 0; mode < 3; ++mode) {
            if (mode == 2 && S > 49152) continue;
            float best = 1e9;
            for (int rep = 0; rep < 4; ++rep) {
                CK(cudaEventRecord(e0));
                if (mode == 0) ell_gather<0><<<148 * 8, 256>>>(didx, rows, K4, dx, S, dy);
                if (mode == 1) ell_gather<1><<<148 * 8, 256>>>(didx, rows, K4, dx, S, dy);
                if (mode == 2) ell_gather<2><<<148, 1024, S * 4>>>(didx, rows, K4, dx, S, dy);
                CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
                float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); if (rep && ms < best) best = ms;
            }
            CK(cudaGetLastError());
            printf("{\"probe\":\"gather\",\"dist\":\"%s\",\"S\":%d,\"mode\":%d,\"ms\":%.3f,\"idx_GBps\":%.1f,\"Ggather_s\":%.1f}\n",
                   dist ? "skew" : "uniform", S, mode, best, nidx * 4 / best / 1e6, nidx / best / 1e6);
        }
    }
    return 0;
}
