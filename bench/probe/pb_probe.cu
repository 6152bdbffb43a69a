// pb_probe.cu -- feasibility probe (not the product): a gather-free two-phase SpMV.
//
// Phase 1 (expand), one CTA per column chunk of one row group: entries of the chunk in CSC order
// read x[col0 + colrel] (a narrow, near-sequential window: L1 hits, no random L2 gathers), form
// a*x and place it in shared memory at a precomputed position (entries grouped by row bin), then
// flush each (chunk, bin) run contiguously into the group's partial buffer (kept L2-resident).
// Phase 2 (reduce), one CTA per row bin: the bin's region of partials is copied into shared
// memory, then every row sums its partials in a fixed order (thread per row over 32-row slabs
// stored column-major, or warp per row with a fixed shuffle tree for long rows): deterministic.
#include <cuda_runtime.h>
#include <stdint.h>

struct Chunk { int64_t e0; int32_t n, col0, run0, nrun; };            // 24 B
struct Run { int32_t start, len; int64_t goff; };                      // 16 B
struct Bin { int64_t roff; int32_t rlen, row0, nrows, slab0, nslab, pad; };
struct Slab { int64_t poff; int32_t w, mode; };                        // mode 0: ELL, 1: warp per row

__device__ __forceinline__ uint64_t pol_last() {
    uint64_t p; asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p)); return p;
}
__device__ __forceinline__ void st_last(float* a, float v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" :: "l"(a), "f"(v), "l"(pol) : "memory");
}

template <bool VALUED>
__global__ void __launch_bounds__(1024) pb_expand(const Chunk* __restrict__ chunks, const Run* __restrict__ runs,
                                                 const uint32_t* __restrict__ cd, const float* __restrict__ val,
                                                 const float* __restrict__ x, float* __restrict__ buf) {
    extern __shared__ float stage[];
    const Chunk c = chunks[blockIdx.x];
    const uint32_t* p = cd + c.e0;
    const float* v = VALUED ? val + c.e0 : nullptr;
    const float* xb = x + c.col0;
    for (int i = threadIdx.x; i < c.n; i += 1024) {
        const uint32_t w = __ldcs(p + i);
        float xv = __ldg(xb + (w & 0xffff));
        if (VALUED) xv *= __ldcs(v + i);
        stage[w >> 16] = xv;
    }
    __syncthreads();
    const uint64_t pol = pol_last();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int r = warp; r < c.nrun; r += 32) {
        const Run ru = runs[c.run0 + r];
        for (int k = lane; k < ru.len; k += 32) st_last(buf + ru.goff + k, stage[ru.start + k], pol);
    }
}

__global__ void __launch_bounds__(1024) pb_reduce(const Bin* __restrict__ bins, const Slab* __restrict__ slabs,
                                                 const uint16_t* __restrict__ pos, const int32_t* __restrict__ rowlen,
                                                 const float* __restrict__ buf, float* __restrict__ y) {
    extern __shared__ float reg[];
    const Bin b = bins[blockIdx.x];
    const float* src = buf + b.roff;
    for (int i = threadIdx.x; i < b.rlen; i += 1024) reg[i] = __ldcs(src + i);
    if (threadIdx.x == 0) reg[b.rlen] = 0.0f;                 // padding position -> 0
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int s = warp; s < b.nslab; s += 32) {
        const Slab sl = slabs[b.slab0 + s];
        const int r0 = s * 32;
        if (sl.mode == 0) {
            const uint16_t* pp = pos + sl.poff + lane;
            float acc = 0.0f;
            int k = 0;
            for (; k + 4 <= sl.w; k += 4) {
                const uint16_t q0 = __ldcs(pp + 32 * k), q1 = __ldcs(pp + 32 * (k + 1));
                const uint16_t q2 = __ldcs(pp + 32 * (k + 2)), q3 = __ldcs(pp + 32 * (k + 3));
                acc += reg[q0]; acc += reg[q1]; acc += reg[q2]; acc += reg[q3];
            }
            for (; k < sl.w; ++k) acc += reg[__ldcs(pp + 32 * k)];
            if (r0 + lane < b.nrows) y[b.row0 + r0 + lane] = acc;
        } else {
            // up to 32 rows, each at its own length, row-major
            const uint16_t* pp = pos + sl.poff;
            for (int rr = 0; rr < 32 && r0 + rr < b.nrows; ++rr) {
                const int len = rowlen[b.row0 + r0 + rr];
                float acc = 0.0f;
                for (int k = lane; k < len; k += 32) acc += reg[__ldcs(pp + k)];
                pp += len;
                for (int o = 16; o >= 1; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
                if (lane == 0) y[b.row0 + r0 + rr] = acc;
            }
        }
    }
}

extern "C" {
int pb_setup(int stage_bytes, int region_bytes) {
    cudaError_t e = cudaFuncSetAttribute(pb_expand<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, stage_bytes);
    if (!e) e = cudaFuncSetAttribute(pb_expand<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, stage_bytes);
    if (!e) e = cudaFuncSetAttribute(pb_reduce, cudaFuncAttributeMaxDynamicSharedMemorySize, region_bytes);
    return (int)e;
}
// one SpMV: for each group g: expand chunks [gc[g], gc[g+1]), reduce bins [gb[g], gb[g+1])
int pb_run(int G, const int32_t* gc, const int32_t* gb, const void* chunks, const void* runs,
           const uint32_t* cd, const float* val, const float* x, float* buf, const void* bins,
           const void* slabs, const uint16_t* pos, const int32_t* rowlen, float* y, int stage_bytes, int region_bytes,
           void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    for (int g = 0; g < G; ++g) {
        const int nc = gc[g + 1] - gc[g], nb = gb[g + 1] - gb[g];
        const Chunk* ch = (const Chunk*)chunks + gc[g];
        if (nc > 0) {
            if (val) pb_expand<true><<<nc, 1024, stage_bytes, st>>>(ch, (const Run*)runs, cd, val, x, buf);
            else pb_expand<false><<<nc, 1024, stage_bytes, st>>>(ch, (const Run*)runs, cd, val, x, buf);
        }
        if (nb > 0) pb_reduce<<<nb, 1024, region_bytes, st>>>((const Bin*)bins + gb[g], (const Slab*)slabs, pos, rowlen, buf, y);
    }
    return (int)cudaGetLastError();
}
}
