// Hardware probe: random x gathers through the TMA engine (cp.async.bulk.tensor.2d ...
// tile::gather4, sm_100a) versus plain ld.global gathers, same index stream.  Question: does the
// tensor-copy path deliver more random 32-byte rows per SM-cycle than the L1 -> L2 request path
// (which saturates near 1 sector request per SM-cycle, profiles/README.md)?
// Not part of the product path.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe3 probe3.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t* b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mb_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t par) {
    uint32_t ok = 0;
    while (!ok) {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
                     "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(sa(b)), "r"(par) : "memory");
    }
}
__device__ __forceinline__ void gather4(void* dst, const CUtensorMap* tm, int4 r, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
        ::"r"(sa(dst)), "l"(tm), "r"(0), "r"(r.x), "r"(r.y), "r"(r.z), "r"(r.w), "r"(sa(bar)) : "memory");
}

constexpr int kST = 4;      // ring stages per warp
constexpr int kRowB = 32;   // bytes per gathered row (one sector: 8 floats)

// Every warp: per stage, 32 lanes each issue one gather4 (4 rows) = 128 rows = 4 KB.
template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1) tma_gather(const __grid_constant__ CUtensorMap tm, const int4* __restrict__ idx,
                                                            int64_t n4, float* out) {
    extern __shared__ __align__(128) unsigned char sm[];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char* ring = sm + (size_t)w * kST * 32 * 4 * kRowB;
    __shared__ uint64_t bars[WARPS][kST];
    if (lane == 0) for (int s = 0; s < kST; ++s) mb_init(&bars[w][s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    const int64_t gw = (int64_t)blockIdx.x * WARPS + w, G = (int64_t)gridDim.x * WARPS;
    // batches of 32 int4 (one per lane) handled by warp gw: b = gw, gw + G, ...
    const int64_t nb = n4 / 32;
    auto issue = [&](int64_t b, int s) {
        if (lane == 0) mb_expect(&bars[w][s], 32 * 4 * kRowB);
        __syncwarp();
        int4 r = __ldcs(idx + b * 32 + lane);
        gather4(ring + ((size_t)s * 32 + lane) * 4 * kRowB, &tm, r, &bars[w][s]);
    };
    int64_t b = gw;
    for (int s = 0; s < kST && b + s * G < nb; ++s) issue(b + s * G, s);
    float acc = 0.f;
    uint32_t phase = 0;
    int s = 0;
    for (; b < nb; b += G) {
        mb_wait(&bars[w][s], phase);
        const float* v = reinterpret_cast<const float*>(ring + (size_t)s * 32 * 4 * kRowB);
        #pragma unroll
        for (int q = 0; q < 4; ++q) acc += v[(lane * 4 + q) * 8 + (lane & 7)];
        __syncwarp();
        const int64_t bn = b + kST * G;
        if (bn < nb) issue(bn, s);
        if (++s == kST) { s = 0; phase ^= 1; }
    }
    if (acc == 1.2345f) out[0] = acc;
}

// Same rows through ld.global: lane gathers 4 rows' element (lane & 7).
__global__ void ldg_gather(const float* __restrict__ x, const int4* __restrict__ idx, int64_t n4, float* out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, st = (int64_t)gridDim.x * blockDim.x;
    float acc = 0.f;
    for (; i < n4; i += st) {
        int4 r = __ldcs(idx + i);
        const int e = threadIdx.x & 7;
        acc += x[(int64_t)r.x * 8 + e] + x[(int64_t)r.y * 8 + e] + x[(int64_t)r.z * 8 + e] + x[(int64_t)r.w * 8 + e];
    }
    if (acc == 1.2345f) out[0] = acc;
}

static uint64_t sm64(uint64_t z) { z += 0x9E3779B97F4A7C15ull; z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull; z = (z ^ (z >> 27)) * 0x94D049BB133111EBull; return z ^ (z >> 31); }

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int WARPS>
static void run_tma(const CUtensorMap& tm, const int4* d_idx, int64_t n4, float* dout, int64_t rows, const char* dist) {
    const size_t smem = (size_t)WARPS * kST * 32 * 4 * kRowB;
    CK(cudaFuncSetAttribute(tma_gather<WARPS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int nb = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, tma_gather<WARPS>, WARPS * 32, smem));
    cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        CK(cudaEventRecord(e0));
        tma_gather<WARPS><<<148 * nb, WARPS * 32, smem>>>(tm, d_idx, n4, dout);
        CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaGetLastError());
        float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); if (ms < best) best = ms;
    }
    printf("{\"probe\":\"tma_gather4\",\"dist\":\"%s\",\"rows\":%lld,\"warps\":%d,\"ctas_per_sm\":%d,\"ms\":%.3f,\"Grows_s\":%.1f}\n",
           dist, (long long)rows, WARPS, nb, best, n4 * 4 / best / 1e6);
}

int main() {
    EncodeFn enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
    float* dout; CK(cudaMalloc(&dout, 4));
    const int64_t G4 = 1 << 24;                      // 16M gather4 = 64M rows per pass
    int4* d_idx; CK(cudaMalloc(&d_idx, G4 * 16));
    for (int64_t rows : {4847571LL / 8 + 1, 41291594LL / 8 + 1}) {
        float* x; CK(cudaMalloc(&x, rows * kRowB)); CK(cudaMemset(x, 0, rows * kRowB));
        CUtensorMap tm;
        cuuint64_t dims[2] = {8, (cuuint64_t)rows};
        cuuint64_t strides[1] = {kRowB};
        cuuint32_t box[2] = {8, 1};
        cuuint32_t es[2] = {1, 1};
        CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, x, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) { printf("{\"error\":\"encode %d\"}\n", (int)r); return 1; }
        for (int skew = 0; skew < 2; ++skew) {
            std::vector<int32_t> h(G4 * 4);
            for (int64_t i = 0; i < G4 * 4; ++i) {
                uint64_t z = sm64(i * 7 + skew);
                double u = (z >> 11) * (1.0 / 9007199254740992.0);
                h[i] = skew ? (int32_t)(rows * u * u * u * u) : (int32_t)(z % rows);
                if (h[i] >= rows) h[i] = (int32_t)rows - 1;
            }
            CK(cudaMemcpy(d_idx, h.data(), G4 * 16, cudaMemcpyHostToDevice));
            const char* dist = skew ? "skew_u4" : "uniform";
            cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
            float best = 1e30f;
            for (int rep = 0; rep < 5; ++rep) {
                CK(cudaEventRecord(e0));
                ldg_gather<<<148 * 8, 256>>>(x, d_idx, G4, dout);
                CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
                float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); if (ms < best) best = ms;
            }
            printf("{\"probe\":\"ldg_gather\",\"dist\":\"%s\",\"rows\":%lld,\"ms\":%.3f,\"Grows_s\":%.1f}\n", dist,
                   (long long)rows, best, G4 * 4 / best / 1e6);
            run_tma<4>(tm, d_idx, G4, dout, rows, dist);
            run_tma<8>(tm, d_idx, G4, dout, rows, dist);
            run_tma<16>(tm, d_idx, G4, dout, rows, dist);
        }
        CK(cudaFree(x));
    }
    return 0;
}
