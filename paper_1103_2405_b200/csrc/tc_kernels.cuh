// tc_kernels.cuh -- sm_100a TILE-COMPOSITE SpMV kernels.
//
// One launch per tile, tiles in ascending order ("restart a kernel for each tile";
// the next tile must see this tile's y writes).  Inside a launch every warp runs whole workloads
// (Solution 3, L88: "each workload is assigned to a warp of threads"), statically round-robin over
// a persistent grid (the workloads are balanced by construction, ~WL slots each).
//
//   row-major workload (w >= h, CSR-vector, L80-L82, L94): `lpr` lanes per row (the smallest
//     power of two covering w/4 int4 groups, at most 32), 32/lpr rows per warp step, 128-bit
//     streaming loads of col/val, shuffle-xor reduction inside each lane group.
//   column-major workload (w < h, ELL, L84, L94): thread per row over 32-row slabs, slots
//     k-interleaved by kvec in {4,2,1} so each lane issues 128/64/32-bit coalesced loads; the
//     whole workload is one linear stream of 32*kvec-slot units, a row ends every w/kvec units.
//   split chunk (rows longer than WL, reading R21): row-major, h = 1; partial stored, the last
//     arriving chunk sums all partials in chunk order (deterministic) and writes the row.
//
// x: dense tiles stage their x segment in shared memory once per CTA (Solution 1, L56-L58: the
// segment "stays" on chip until the tile finishes); the remainder gathers through the read-only
// path (L1/L2; x fits in the 126 MB L2 at the single-GPU configs) -- the paper's remainder is
// likewise modelled "without using the texture cache" (L160).
// col/val are streamed once with evict-first hints so they do not push x out of L2.
// y: within a tile each row has one writer; a row's first tile stores, later tiles add (FLAG_ACC);
// the tile order is fixed, so results are bitwise deterministic (no atomics on y).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "plan.h"

namespace tc {

constexpr int kThreads = 768;            // 24 warps per CTA: one CTA per SM at <= 80 registers (no spills)
constexpr int kWarps = kThreads / 32;

struct TileArgs {
    const WlDesc* desc;
    int64_t wl_begin, wl_end;
    const int32_t* col;       // slot columns (tile-relative)
    const float* val;         // slot values (nullptr: pattern)
    const uint32_t* row_id;
    const float* x;           // x' + col_lo: tile-relative base of the relabelled x
    int32_t width;            // tile width = padding sentinel
    const int32_t* split;     // [n_split][3]
    float* partials;          // [n_chunks]
    int32_t* counters;        // [n_split], zero between launches
};

__device__ __forceinline__ int4 ld_stream_i4(const int32_t* p) {
    return __ldcs(reinterpret_cast<const int4*>(p));
}
__device__ __forceinline__ float4 ld_stream_f4(const float* p) {
    return __ldcs(reinterpret_cast<const float4*>(p));
}
__device__ __forceinline__ int2 ld_stream_i2(const int32_t* p) {
    return __ldcs(reinterpret_cast<const int2*>(p));
}
__device__ __forceinline__ float2 ld_stream_f2(const float* p) {
    return __ldcs(reinterpret_cast<const float2*>(p));
}

template <bool STAGED>
struct XSrc {
    const float* g;     // global base (tile-relative)
    const float* s;     // shared base
    int32_t width;
    __device__ __forceinline__ float operator()(int32_t c) const {
        if (c == width) return 0.0f;                  // padding slot (sentinel, reading R16)
        if (STAGED) return s[c];
        return __ldg(g + c);
    }
};

// one vector of KV slots: load cols (+vals), gather x, return the partial dot product
template <int KV, bool VALUED>
struct Unit;

template <bool VALUED>
struct Unit<4, VALUED> {
    int4 c; float4 v;
    __device__ __forceinline__ void load(const int32_t* col, const float* val, int s) {
        c = ld_stream_i4(col + s);
        if (VALUED) v = ld_stream_f4(val + s);
    }
    template <class X>
    __device__ __forceinline__ float dot(const X& x) const {
        float x0 = x(c.x), x1 = x(c.y), x2 = x(c.z), x3 = x(c.w);
        if (VALUED) return fmaf(v.x, x0, fmaf(v.y, x1, fmaf(v.z, x2, v.w * x3)));
        return (x0 + x1) + (x2 + x3);
    }
};
template <bool VALUED>
struct Unit<2, VALUED> {
    int2 c; float2 v;
    __device__ __forceinline__ void load(const int32_t* col, const float* val, int s) {
        c = ld_stream_i2(col + s);
        if (VALUED) v = ld_stream_f2(val + s);
    }
    template <class X>
    __device__ __forceinline__ float dot(const X& x) const {
        float x0 = x(c.x), x1 = x(c.y);
        if (VALUED) return fmaf(v.x, x0, v.y * x1);
        return x0 + x1;
    }
};
template <bool VALUED>
struct Unit<1, VALUED> {
    int32_t c; float v;
    __device__ __forceinline__ void load(const int32_t* col, const float* val, int s) {
        c = __ldcs(col + s);
        if (VALUED) v = __ldcs(val + s);
    }
    template <class X>
    __device__ __forceinline__ float dot(const X& x) const {
        float x0 = x(c);
        if (VALUED) return v * x0;
        return x0;
    }
};

// Row write with split-chunk combine.  Epi::write(entry, value) stores / accumulates / applies
// the fused epilogue.  Called by exactly one lane per row.
template <class Epi>
__device__ __forceinline__ void finish_split(const TileArgs& a, const WlDesc& d, uint32_t ent,
                                             float v, Epi& epi) {
    const int32_t* sp = a.split + 3 * d.split_id;
    const int32_t nch = __ldg(sp + 1), pbase = __ldg(sp + 2);
    a.partials[pbase + d.chunk] = v;
    __threadfence();
    int32_t t = atomicAdd(a.counters + d.split_id, 1);
    if (t == nch - 1) {
        __threadfence();
        float s = 0.0f;
        for (int32_t c = 0; c < nch; ++c) s += __ldcg(a.partials + pbase + c);
        a.counters[d.split_id] = 0;                   // ready for the next launch
        epi.write(ent, s);
    }
}

template <bool VALUED, class X, class Epi>
__device__ __forceinline__ void run_rm(const TileArgs& a, const WlDesc& d, const X& x, Epi& epi,
                                       int lane) {
    const int w4 = d.w >> 2;                          // int4 groups per row
    const int lpr = w4 >= 32 ? 32 : (w4 <= 1 ? 1 : (1 << (32 - __clz(w4 - 1))));
    const int lg = __ffs(lpr) - 1;
    const int rps = 32 >> lg;
    const int sub = lane >> lg, sl = lane & (lpr - 1);
    for (int r0 = 0; r0 < d.h; r0 += rps) {
        const int r = r0 + sub;
        const bool act = r < d.h;
        uint32_t ent = (act && sl == 0) ? __ldg(a.row_id + d.row_base + r) : PAD_ROW;
        const int64_t base = d.off + (int64_t)r * d.w;
        const int32_t* cb = a.col + base;
        const float* vb = VALUED ? a.val + base : nullptr;
        const int qend = act ? w4 : 0;
        float acc = 0.0f;
        int q = sl;
        for (; q + lpr < qend; q += 2 * lpr) {
            Unit<4, VALUED> u0, u1;
            u0.load(cb, vb, 4 * q);
            u1.load(cb, vb, 4 * (q + lpr));
            acc += u0.dot(x) + u1.dot(x);
        }
        if (q < qend) {
            Unit<4, VALUED> u0;
            u0.load(cb, vb, 4 * q);
            acc += u0.dot(x);
        }
        for (int o = lpr >> 1; o >= 1; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (act && sl == 0) {
            if (d.kind == KIND_SPLIT) finish_split(a, d, ent, acc, epi);
            else epi.write(ent, acc);
        }
    }
}

template <int KV, bool VALUED, class X, class Epi>
__device__ __forceinline__ void run_cm(const TileArgs& a, const WlDesc& d, const X& x, Epi& epi,
                                       int lane) {
    constexpr int UN = KV == 4 ? 2 : 4;               // 32-64 bytes in flight per lane (valued)
    const int nk = d.w / KV;                          // units per slab
    const int slabs = d.h >> 5;
    const int total = slabs * nk;                     // units (< 2^31: WL-bounded workloads)
    const uint32_t* rid = a.row_id + d.row_base + lane;
    const int32_t* cb = a.col + d.off + lane * KV;
    const float* vb = VALUED ? a.val + d.off + lane * KV : nullptr;
    int kk = 0, s = 0;
    uint32_t ent = slabs > 0 ? __ldg(rid) : PAD_ROW;
    float acc = 0.0f;
    for (int u0 = 0; u0 < total; u0 += UN) {
        Unit<KV, VALUED> u[UN];
        #pragma unroll
        for (int j = 0; j < UN; ++j)
            if (u0 + j < total) u[j].load(cb, vb, (u0 + j) * (32 * KV));
        #pragma unroll
        for (int j = 0; j < UN; ++j) {
            if (u0 + j < total) {
                acc += u[j].dot(x);
                if (++kk == nk) {
                    if (ent != PAD_ROW) epi.write(ent, acc);
                    acc = 0.0f; kk = 0; ++s;
                    ent = s < slabs ? __ldg(rid + 32 * s) : PAD_ROW;
                }
            }
        }
    }
}

// zero-length rows (remainder tile): every row of every slab gets value 0
template <class Epi>
__device__ __forceinline__ void run_zero(const TileArgs& a, const WlDesc& d, Epi& epi, int lane) {
    for (int r = lane; r < d.h; r += 32) {
        uint32_t ent = __ldg(a.row_id + d.row_base + r);
        if (ent != PAD_ROW) epi.write(ent, 0.0f);
    }
}

template <bool STAGED, bool VALUED, class Epi>
__global__ void __launch_bounds__(kThreads, 1) tc_spmv_tile(TileArgs a, Epi epi_in) {
    extern __shared__ float xs[];
    Epi epi = epi_in;
    if (!epi.begin()) return;                         // iteration loop already converged
    if (STAGED) {
        // stage the tile's x segment once per CTA (float4 where aligned)
        const float* src = a.x;
        const int n = a.width;
        const int head = (int)((4 - ((reinterpret_cast<uintptr_t>(src) >> 2) & 3)) & 3);
        const int h = head < n ? head : n;
        for (int i = threadIdx.x; i < h; i += kThreads) xs[i] = __ldg(src + i);
        const int n4 = (n - h) >> 2;
        const float4* s4 = reinterpret_cast<const float4*>(src + h);
        for (int i = threadIdx.x; i < n4; i += kThreads) {
            float4 v = __ldg(s4 + i);
            xs[h + 4 * i] = v.x; xs[h + 4 * i + 1] = v.y; xs[h + 4 * i + 2] = v.z; xs[h + 4 * i + 3] = v.w;
        }
        for (int i = h + 4 * n4 + threadIdx.x; i < n; i += kThreads) xs[i] = __ldg(src + i);
        __syncthreads();
    }
    XSrc<STAGED> x{a.x, xs, a.width};
    const int lane = threadIdx.x & 31;
    const int64_t gw = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
    const int64_t G = (int64_t)gridDim.x * kWarps;
    for (int64_t j = a.wl_begin + gw; j < a.wl_end; j += G) {
        const int4* dp = reinterpret_cast<const int4*>(a.desc + j);
        int4 d0 = __ldg(dp), d1 = __ldg(dp + 1);
        WlDesc d;
        d.off = (int64_t)(((uint64_t)(uint32_t)d0.y << 32) | (uint32_t)d0.x);
        d.row_base = d0.z; d.w = d0.w; d.h = d1.x;
        d.kind = (uint8_t)(d1.y & 0xff); d.kvec = (uint8_t)((d1.y >> 8) & 0xff);
        d.split_id = d1.z; d.chunk = d1.w;
        if (d.kind != KIND_CM) {
            run_rm<VALUED>(a, d, x, epi, lane);
        } else if (d.w == 0) {
            run_zero(a, d, epi, lane);
        } else if (d.kvec == 4) {
            run_cm<4, VALUED>(a, d, x, epi, lane);
        } else if (d.kvec == 2) {
            run_cm<2, VALUED>(a, d, x, epi, lane);
        } else {
            run_cm<1, VALUED>(a, d, x, epi, lane);
        }
    }
    epi.end();
}

// y = A x epilogue-free writer
struct EpiStore {
    float* y;
    __device__ __forceinline__ bool begin() { return true; }
    __device__ __forceinline__ void end() {}
    __device__ __forceinline__ void write(uint32_t ent, float v) {
        const uint32_t r = ent & ROW_MASK;
        if (ent & FLAG_ACC) v += y[r];
        y[r] = v;
    }
};

}  // namespace tc
