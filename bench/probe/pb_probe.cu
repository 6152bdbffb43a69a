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

#include "tc_async.cuh"

struct Chunk { int64_t e0; int32_t n, col0, run0, nrun; };            // 24 B
struct Run { int32_t start, len; int64_t goff; };                      // 16 B
struct Bin { int64_t roff; int32_t rlen, row0, nrows, slab0, nslab, nheavy; int64_t hoff; int32_t plen, pad2; };
struct Slab { int64_t poff; int32_t w, mode; };                        // mode 0: ELL, 1: warp per row

__device__ __forceinline__ uint64_t pol_last() {
    uint64_t p; asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p)); return p;
}
__device__ __forceinline__ void st_last(float* a, float v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" :: "l"(a), "f"(v), "l"(pol) : "memory");
}

#ifndef PB_FLAT
#define PB_FLAT 1
#endif
#ifndef PB_POS_SMEM
#define PB_POS_SMEM 0
#endif
#if PB_POS_SMEM
#define LDP(p) (*(p))
#else
#define LDP(p) __ldcs(p)
#endif
#ifndef PB_CMAX
#define PB_CMAX 16384
#endif
#ifndef PB_ET
#define PB_ET 512
#endif
#ifndef PB_RT
#define PB_RT 512
#endif
__device__ const uint16_t* g_rid;                          // PB_FLAT == 2: run index per stage position
template <bool VALUED>
__global__ void __launch_bounds__(PB_ET, 2) pb_expand(const Chunk* __restrict__ chunks, const Run* __restrict__ runs,
                                                      const uint32_t* __restrict__ cd, const float* __restrict__ val,
                                                      const float* __restrict__ x, float* __restrict__ buf) {
    extern __shared__ float stage[];
    const Chunk c = chunks[blockIdx.x];
    const uint32_t* p = cd + c.e0;
    const float* v = VALUED ? val + c.e0 : nullptr;
    const float* xb = x + c.col0;
#if PB_FLAT
    // run table of this chunk in shared memory: goff (8 B) then start (4 B) per run
    long long* rg = reinterpret_cast<long long*>(stage + PB_CMAX);
    int* rs = reinterpret_cast<int*>(rg + c.nrun);
    for (int r = threadIdx.x; r < c.nrun; r += PB_ET) {
        const Run ru = runs[c.run0 + r];
        rs[r] = ru.start;
        rg[r] = ru.goff;
    }
#endif
    constexpr int U = 8;
    for (int i0 = threadIdx.x; i0 < c.n; i0 += PB_ET * U) {
        uint32_t w[U];
        float a[U], xv[U];
        #pragma unroll
        for (int j = 0; j < U; ++j) {
            const int i = i0 + j * PB_ET;
            w[j] = i < c.n ? __ldcs(p + i) : 0xffffffffu;
            if (VALUED) a[j] = i < c.n ? __ldcs(v + i) : 0.0f;
        }
        #pragma unroll
        for (int j = 0; j < U; ++j) xv[j] = w[j] != 0xffffffffu ? __ldg(xb + (w[j] & 0xffff)) : 0.0f;
        #pragma unroll
        for (int j = 0; j < U; ++j)
            if (w[j] != 0xffffffffu) stage[w[j] >> 16] = VALUED ? a[j] * xv[j] : xv[j];
    }
    __syncthreads();
    const uint64_t pol = pol_last();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // flat flush: warp w stores stage positions [q0, q0 + 32) for q0 = 32w, 32w + PB_ET, ...; the
    // runs (sorted by stage start) are found with one ballot-free step per 32 positions: lanes hold
    // a window of 32 run descriptors; runs starting inside the step set bits of a mask (redux.or),
    // and lane i's run is the window base + popc(mask & lanes <= i) - 1 (+ the run open at q0)
#if PB_FLAT == 2
    // static run index of every stage position (2 B, coalesced): destination without a search
    for (int q = threadIdx.x; q < c.n; q += PB_ET) {
        const int r = __ldcs(g_rid + c.e0 + q);
        st_last(buf + rg[r] + (q - rs[r]), stage[q], pol);
    }
#elif PB_FLAT
    const int L = ((c.n + PB_ET / 32 - 1) / (PB_ET / 32) + 31) & ~31;   // positions per warp (multiple of 32)
    const int q_beg = warp * L, q_end = min(c.n, q_beg + L);
    if (q_beg < q_end) {
        int lo = 0, hi = c.nrun - 1;                               // run containing q_beg
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (rs[mid] <= q_beg) lo = mid; else hi = mid - 1;
        }
        for (int q0 = q_beg; q0 < q_end; q0 += 32) {
            const bool have = lo + lane < c.nrun;
            const int mys = have ? rs[lo + lane] : 0x7fffffff;
            const int d = mys - q0;                                // run lo + lane starts at offset d
            const unsigned bit = (lane > 0 && have && d >= 0 && d < 32) ? (1u << d) : 0u;
            const unsigned M = __reduce_or_sync(0xffffffffu, bit);
            const int j = __popc(M & (0xffffffffu >> (31 - lane)));   // runs started in [q0, q0 + lane]
            const int st0 = __shfl_sync(0xffffffffu, mys, j);
            const long long go = rg[lo + j];
            const int q = q0 + lane;
            if (q < q_end) st_last(buf + go + (q - st0), stage[q], pol);
            lo += __popc(M);
        }
    }
#else
    // each warp takes 32 runs at a time: one descriptor per lane (a single load round trip),
    // then the warp stores the runs one after another (stores do not wait)
    for (int r0 = warp * 32; r0 < c.nrun; r0 += PB_ET) {
        Run my{0, 0, 0};
        if (r0 + lane < c.nrun) my = runs[c.run0 + r0 + lane];
        const int cnt = min(32, c.nrun - r0);
        for (int j = 0; j < cnt; ++j) {
            const int st0 = __shfl_sync(0xffffffffu, my.start, j);
            const int len = __shfl_sync(0xffffffffu, my.len, j);
            const long long go = __shfl_sync(0xffffffffu, (long long)my.goff, j);
            for (int k = lane; k < len; k += 32) st_last(buf + go + k, stage[st0 + k], pol);
        }
    }
#endif
}

__global__ void __launch_bounds__(PB_RT, 2) pb_reduce(const Bin* __restrict__ bins, const Slab* __restrict__ slabs,
                                                  const uint16_t* __restrict__ pos, const int64_t* __restrict__ rcum,
                                                  const float* __restrict__ buf, float* __restrict__ y) {
    extern __shared__ float reg[];
    __shared__ float wsum[PB_RT / 32];
    const Bin b = bins[blockIdx.x];
    const float* src = buf + b.roff;
    {   // regions start 16-byte aligned (builder); float4 loads, four in flight per thread
        const float4* s4 = reinterpret_cast<const float4*>(src);
        float4* d4 = reinterpret_cast<float4*>(reg);
        const int n4 = (b.rlen + 3) >> 2;
        for (int i0 = threadIdx.x; i0 < n4; i0 += PB_RT * 4) {
            float4 t[4];
            #pragma unroll
            for (int j = 0; j < 4; ++j) if (i0 + j * PB_RT < n4) t[j] = __ldcs(s4 + i0 + j * PB_RT);
            #pragma unroll
            for (int j = 0; j < 4; ++j) if (i0 + j * PB_RT < n4) d4[i0 + j * PB_RT] = t[j];
        }
    }
#if PB_POS_SMEM
    // the bin's position block (heavy rows, then light slabs; 16-byte aligned, padded to 8) too
    uint16_t* ps = reinterpret_cast<uint16_t*>(reg + ((b.rlen + 8 + 3) & ~3));
    {
        const uint4* s8 = reinterpret_cast<const uint4*>(pos + b.hoff);
        uint4* d8 = reinterpret_cast<uint4*>(ps);
        const int n8 = b.plen >> 3;
        for (int i0 = threadIdx.x; i0 < n8; i0 += PB_RT * 4) {
            uint4 t[4];
            #pragma unroll
            for (int j = 0; j < 4; ++j) if (i0 + j * PB_RT < n8) t[j] = __ldcs(s8 + i0 + j * PB_RT);
            #pragma unroll
            for (int j = 0; j < 4; ++j) if (i0 + j * PB_RT < n8) d8[i0 + j * PB_RT] = t[j];
        }
    }
    const uint16_t* pbase = ps - b.hoff;                      // pbase[global pos index]
#else
    const uint16_t* pbase = pos;
#endif
    __syncthreads();
    if (threadIdx.x == 0) reg[b.rlen] = 0.0f;                 // padding position -> 0
    __syncthreads();
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // heavy rows (a prefix of the bin: rows are length-sorted), positions row-major at hoff
    const int64_t c0 = rcum[b.row0];
    int r = 0;
    for (; r < b.nheavy; ++r) {                                 // giant rows: the whole CTA, fixed tree
        const int64_t o = rcum[b.row0 + r] - c0, len = rcum[b.row0 + r + 1] - rcum[b.row0 + r];
        if (len < 4096) break;
        const uint16_t* pp = pbase + b.hoff + o;
        float acc = 0.0f;
        for (int64_t k = threadIdx.x; k < len; k += PB_RT) acc += reg[LDP(pp + k)];
        for (int q = 16; q >= 1; q >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, q);
        if (lane == 0) wsum[warp] = acc;
        __syncthreads();
        if (warp == 0) {
            float v = lane < PB_RT / 32 ? wsum[lane] : 0.0f;
            for (int q = 16; q >= 1; q >>= 1) v += __shfl_xor_sync(0xffffffffu, v, q);
            if (lane == 0) y[b.row0 + r] = v;
        }
        __syncthreads();
    }
    for (int rr = r + warp; rr < b.nheavy; rr += PB_RT / 32) {          // warp per row
        const int64_t o = rcum[b.row0 + rr] - c0, len = rcum[b.row0 + rr + 1] - rcum[b.row0 + rr];
        const uint16_t* pp = pbase + b.hoff + o;
        float acc = 0.0f;
        for (int64_t k = lane; k < len; k += 32) acc += reg[LDP(pp + k)];
        for (int q = 16; q >= 1; q >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, q);
        if (lane == 0) y[b.row0 + rr] = acc;
    }
    // light rows: 32-row ELL slabs after the heavy prefix, thread per row
    for (int s = warp; s < b.nslab; s += PB_RT / 32) {
        const Slab sl = slabs[b.slab0 + s];
        const int rl = b.nheavy + s * 32 + lane;
        const uint16_t* pp = pbase + sl.poff + lane;
        float acc = 0.0f;
        int k = 0;
        for (; k + 8 <= sl.w; k += 8) {
            uint16_t q[8];
            #pragma unroll
            for (int j = 0; j < 8; ++j) q[j] = LDP(pp + 32 * (k + j));
            #pragma unroll
            for (int j = 0; j < 8; ++j) acc += reg[q[j]];
        }
        for (; k < sl.w; ++k) acc += reg[LDP(pp + 32 * k)];
        if (rl < b.nrows) y[b.row0 + rl] = acc;
    }
}


// persistent reduce: each CTA walks bins blockIdx.x, + gridDim.x, ...; the next bin's region is
// bulk-copied (cp.async.bulk, TMA 1-D) into the other shared buffer while this one is summed
__device__ __forceinline__ void reduce_bin(const Bin& b, const Slab* __restrict__ slabs,
                                           const uint16_t* __restrict__ pos, const int64_t* __restrict__ rcum,
                                           const float* reg, float* __restrict__ y, float* wsum) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t c0 = rcum[b.row0];
    int r = 0;
    for (; r < b.nheavy; ++r) {
        const int64_t o = rcum[b.row0 + r] - c0, len = rcum[b.row0 + r + 1] - rcum[b.row0 + r];
        if (len < 4096) break;
        const uint16_t* pp = pos + b.hoff + o;
        float acc = 0.0f;
        for (int64_t k = threadIdx.x; k < len; k += PB_RT) acc += reg[__ldcs(pp + k)];
        for (int q = 16; q >= 1; q >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, q);
        if (lane == 0) wsum[warp] = acc;
        __syncthreads();
        if (warp == 0) {
            float v = lane < PB_RT / 32 ? wsum[lane] : 0.0f;
            for (int q = 16; q >= 1; q >>= 1) v += __shfl_xor_sync(0xffffffffu, v, q);
            if (lane == 0) y[b.row0 + r] = v;
        }
        __syncthreads();
    }
    for (int rr = r + warp; rr < b.nheavy; rr += PB_RT / 32) {
        const int64_t o = rcum[b.row0 + rr] - c0, len = rcum[b.row0 + rr + 1] - rcum[b.row0 + rr];
        const uint16_t* pp = pos + b.hoff + o;
        float acc = 0.0f;
        for (int64_t k = lane; k < len; k += 32) acc += reg[__ldcs(pp + k)];
        for (int q = 16; q >= 1; q >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, q);
        if (lane == 0) y[b.row0 + rr] = acc;
    }
    for (int s = warp; s < b.nslab; s += PB_RT / 32) {
        const Slab sl = slabs[b.slab0 + s];
        const int rl = b.nheavy + s * 32 + lane;
        const uint16_t* pp = pos + sl.poff + lane;
        float acc = 0.0f;
        int k = 0;
        for (; k + 8 <= sl.w; k += 8) {
            uint16_t q[8];
            #pragma unroll
            for (int j = 0; j < 8; ++j) q[j] = __ldcs(pp + 32 * (k + j));
            #pragma unroll
            for (int j = 0; j < 8; ++j) acc += reg[q[j]];
        }
        for (; k < sl.w; ++k) acc += reg[__ldcs(pp + 32 * k)];
        if (rl < b.nrows) y[b.row0 + rl] = acc;
    }
}

#ifndef PB_PIPE_CTAS
#define PB_PIPE_CTAS 1
#endif
__global__ void __launch_bounds__(PB_RT, PB_PIPE_CTAS) pb_reduce_pipe(const Bin* __restrict__ bins, int nbins, int buf_floats,
                                                       const Slab* __restrict__ slabs, const uint16_t* __restrict__ pos,
                                                       const int64_t* __restrict__ rcum, const float* __restrict__ buf,
                                                       float* __restrict__ y) {
    extern __shared__ __align__(128) float sm[];
    __shared__ __align__(8) uint64_t bar[2];
    __shared__ float wsum[PB_RT / 32];
    float* rb[2] = {sm, sm + buf_floats};
    if (threadIdx.x == 0) { tc::mbar_init(&bar[0], 1); tc::mbar_init(&bar[1], 1); tc::fence_barrier_init(); }
    __syncthreads();
    const uint64_t pol = tc::policy_evict_first();
    auto issue = [&](int j, int k) {
        const Bin b = bins[j];
        const uint32_t bytes = (uint32_t)(((b.rlen + 3) & ~3) * 4);
        tc::mbar_arrive_expect_tx(&bar[k], bytes);
        if (bytes) tc::bulk_g2s(rb[k], buf + b.roff, bytes, &bar[k], pol);
    };
    if (threadIdx.x == 0 && (int)blockIdx.x < nbins) issue(blockIdx.x, 0);
    int i = 0;
    for (int j = blockIdx.x; j < nbins; j += gridDim.x, ++i) {
        const int cur = i & 1;
        if (threadIdx.x == 0 && j + (int)gridDim.x < nbins) { tc::fence_proxy_async_shared(); issue(j + gridDim.x, cur ^ 1); }
        const Bin b = bins[j];
        tc::mbar_wait(&bar[cur], (i >> 1) & 1);
        if (threadIdx.x == 0) rb[cur][b.rlen] = 0.0f;         // padding position -> 0
        __syncthreads();
        reduce_bin(b, slabs, pos, rcum, rb[cur], y, wsum);
        __syncthreads();                                       // buffer free for the copy after next
    }
}

extern "C" {
int pb_set_rid(const uint16_t* rid) { return (int)cudaMemcpyToSymbol(g_rid, &rid, sizeof(rid)); }
int pb_setup(int stage_bytes, int region_bytes) {
    cudaError_t e = cudaFuncSetAttribute(pb_expand<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, stage_bytes);
    if (!e) e = cudaFuncSetAttribute(pb_expand<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, stage_bytes);
    if (!e) e = cudaFuncSetAttribute(pb_reduce, cudaFuncAttributeMaxDynamicSharedMemorySize, region_bytes);
    if (!e) e = cudaFuncSetAttribute(pb_reduce_pipe, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * region_bytes + 256);
    return (int)e;
}
// one SpMV: for each group g: expand chunks [gc[g], gc[g+1]), reduce bins [gb[g], gb[g+1])
// phases 4: expand of group g+1 (stream `stream`) overlaps the reduce of group g (a second
// stream), with two group buffers at buf and buf + buf_stride
int pb_run(int G, int phases, const int32_t* gc, const int32_t* gb, const void* chunks, const void* runs,
           const uint32_t* cd, const float* val, const float* x, float* buf, const void* bins,
           const void* slabs, const uint16_t* pos, const int64_t* rcum, float* y, int stage_bytes, int region_bytes,
           void* stream, long long buf_stride) {
    cudaStream_t st = (cudaStream_t)stream;
    const bool pipe_reduce = phases == 8;
    if (phases == 8) phases = 4;
    if (phases == 4) {
        static cudaStream_t s2 = nullptr;
        static cudaEvent_t ex[64], rd[64], fin;
        if (!s2) {
            cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
            for (int i = 0; i < 64; ++i) { cudaEventCreateWithFlags(&ex[i], cudaEventDisableTiming); cudaEventCreateWithFlags(&rd[i], cudaEventDisableTiming); }
            cudaEventCreateWithFlags(&fin, cudaEventDisableTiming);
        }
        cudaEventRecord(fin, st);
        cudaStreamWaitEvent(s2, fin, 0);
        for (int g = 0; g < G; ++g) {
            float* b = buf + (g & 1) * buf_stride;
            const int nc = gc[g + 1] - gc[g], nb = gb[g + 1] - gb[g];
            const Chunk* ch = (const Chunk*)chunks + gc[g];
            if (g >= 2) cudaStreamWaitEvent(st, rd[g - 2], 0);        // buffer free again
            if (nc > 0) {
                if (val) pb_expand<true><<<nc, PB_ET, stage_bytes, st>>>(ch, (const Run*)runs, cd, val, x, b);
                else pb_expand<false><<<nc, PB_ET, stage_bytes, st>>>(ch, (const Run*)runs, cd, val, x, b);
            }
            cudaEventRecord(ex[g], st);
            cudaStreamWaitEvent(s2, ex[g], 0);
            if (nb > 0) {
                if (pipe_reduce) {
                    static int sms = 0;
                    if (!sms) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
                    const int bf = ((region_bytes / 4) + 31) & ~31;
                    pb_reduce_pipe<<<nb < PB_PIPE_CTAS * sms ? nb : PB_PIPE_CTAS * sms, PB_RT, 2 * bf * 4, s2>>>((const Bin*)bins + gb[g], nb, bf,
                                                                                  (const Slab*)slabs, pos, rcum, b, y);
                } else {
                    pb_reduce<<<nb, PB_RT, region_bytes, s2>>>((const Bin*)bins + gb[g], (const Slab*)slabs, pos, rcum, b, y);
                }
            }
            cudaEventRecord(rd[g], s2);
        }
        cudaEventRecord(fin, s2);
        cudaStreamWaitEvent(st, fin, 0);
        return (int)cudaGetLastError();
    }
    for (int g = 0; g < G; ++g) {
        const int nc = gc[g + 1] - gc[g], nb = gb[g + 1] - gb[g];
        const Chunk* ch = (const Chunk*)chunks + gc[g];
        if (nc > 0 && (phases & 1)) {
            if (val) pb_expand<true><<<nc, PB_ET, stage_bytes, st>>>(ch, (const Run*)runs, cd, val, x, buf);
            else pb_expand<false><<<nc, PB_ET, stage_bytes, st>>>(ch, (const Run*)runs, cd, val, x, buf);
        }
        if (nb > 0 && (phases & 2)) pb_reduce<<<nb, PB_RT, region_bytes, st>>>((const Bin*)bins + gb[g], (const Slab*)slabs, pos, rcum, buf, y);
    }
    return (int)cudaGetLastError();
}
}
