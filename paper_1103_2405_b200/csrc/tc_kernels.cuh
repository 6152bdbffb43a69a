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
#include "tc_async.cuh"

namespace tc {

#ifndef TC_THREADS
#define TC_THREADS 512
#endif
#ifndef TC_RM_UB
#define TC_RM_UB 1         // row major: int4 units per lane per batch
#endif
#ifndef TC_CM_SLOTS_V
#define TC_CM_SLOTS_V 2    // column major, valued: slots per lane per batch
#endif
#ifndef TC_CM_SLOTS_P
#define TC_CM_SLOTS_P 2    // column major, pattern: slots per lane per batch
#endif
#ifndef TC_RM_UB_STAGED
#define TC_RM_UB_STAGED 2
#endif
#ifndef TC_CM_SLOTS_V_STAGED
#define TC_CM_SLOTS_V_STAGED 4
#endif
#ifndef TC_CM_SLOTS_P_STAGED
#define TC_CM_SLOTS_P_STAGED 8
#endif
#ifndef TC_DYN
#define TC_DYN 2           // > 0: the last TC_DYN rounds of workloads are claimed dynamically; 0: static
#endif
#ifndef TC_PF_AHEAD
#define TC_PF_AHEAD 0      // L2 bulk prefetch of a warp's workload: 0 = when it starts, k > 0 =
                           // k workloads ahead, -1 = none.  Measured on c2 (profiles/README.md):
                           // 2 ahead keeps ~77 MB of future slots in L2 and evicts x (955 MB of
                           // DRAM reads per SpMV); at start: 635 MB (algorithmic: 610 MB), -8 % time
#endif
#ifndef TC_X_POLICY
#define TC_X_POLICY 1      // 1: x gathers carry an L2 evict-last policy (x stays resident); -3 %
#endif
#ifndef TC_MINB
#define TC_MINB 2          // minimum resident CTAs per SM (__launch_bounds__)
#endif
constexpr int kDynQ = 32;                // dynamic-schedule claim queues per launch
constexpr int kThreads = TC_THREADS;     // threads per CTA of the classic kernel (one CTA per SM)
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
    uint32_t* sched;          // [kDynQ + 1]: claim queues, CTAs done; zero between launches
    int32_t has_acc;          // rows of this launch may carry FLAG_ACC (not the plan's first tile)
};

// Slot loads: SMEM = false streams from global memory with evict-first (ld.global.cs); SMEM = true
// reads slots the bulk-copy ring already placed in shared memory.
template <bool SMEM> __device__ __forceinline__ int4 ld_i4(const int32_t* p) {
    if (SMEM) return *reinterpret_cast<const int4*>(p);
    return __ldcs(reinterpret_cast<const int4*>(p));
}
template <bool SMEM> __device__ __forceinline__ float4 ld_f4(const float* p) {
    if (SMEM) return *reinterpret_cast<const float4*>(p);
    return __ldcs(reinterpret_cast<const float4*>(p));
}
template <bool SMEM> __device__ __forceinline__ int2 ld_i2(const int32_t* p) {
    if (SMEM) return *reinterpret_cast<const int2*>(p);
    return __ldcs(reinterpret_cast<const int2*>(p));
}
template <bool SMEM> __device__ __forceinline__ float2 ld_f2(const float* p) {
    if (SMEM) return *reinterpret_cast<const float2*>(p);
    return __ldcs(reinterpret_cast<const float2*>(p));
}
template <bool SMEM> __device__ __forceinline__ int32_t ld_i1(const int32_t* p) {
    if (SMEM) return *p;
    return __ldcs(p);
}
template <bool SMEM> __device__ __forceinline__ float ld_f1(const float* p) {
    if (SMEM) return *p;
    return __ldcs(p);
}

template <bool STAGED>
struct XSrc {
    // batch sizes (slots in flight per lane): shared-memory gathers are short-lived, so staged
    // tiles afford deeper batches within the 64-register budget
    static constexpr int kRmUnits = STAGED ? TC_RM_UB_STAGED : TC_RM_UB;
    static constexpr int kCmSlotsV = STAGED ? TC_CM_SLOTS_V_STAGED : TC_CM_SLOTS_V;
    static constexpr int kCmSlotsP = STAGED ? TC_CM_SLOTS_P_STAGED : TC_CM_SLOTS_P;
    const float* g;     // global base (tile-relative)
    const float* s;     // shared base
    int32_t width;
    uint64_t pol = 0;   // TC_X_POLICY: L2 evict-last policy for the gathers
    __device__ __forceinline__ float operator()(int32_t c) const {
        if (c == width) return 0.0f;                  // padding slot (sentinel, reading R16)
        if (STAGED) return s[c];
#if TC_X_POLICY
        float v;
        asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(g + c), "l"(pol));
        return v;
#else
        return __ldg(g + c);
#endif
    }
};

// one vector of KV slots: load cols (+vals), gather x, return the partial dot product
template <int KV, bool VALUED, bool SMEM>
struct Unit;

template <bool VALUED, bool SMEM>
struct Unit<4, VALUED, SMEM> {
    int4 c; float4 v;
    __device__ __forceinline__ void load(const int32_t* col, const float* val, int s) {
        c = ld_i4<SMEM>(col + s);
        if (VALUED) v = ld_f4<SMEM>(val + s);
    }
    template <class X>
    __device__ __forceinline__ float dot(const X& x) const {
        float x0 = x(c.x), x1 = x(c.y), x2 = x(c.z), x3 = x(c.w);
        if (VALUED) return fmaf(v.x, x0, fmaf(v.y, x1, fmaf(v.z, x2, v.w * x3)));
        return (x0 + x1) + (x2 + x3);
    }
};
template <bool VALUED, bool SMEM>
struct Unit<2, VALUED, SMEM> {
    int2 c; float2 v;
    __device__ __forceinline__ void load(const int32_t* col, const float* val, int s) {
        c = ld_i2<SMEM>(col + s);
        if (VALUED) v = ld_f2<SMEM>(val + s);
    }
    template <class X>
    __device__ __forceinline__ float dot(const X& x) const {
        float x0 = x(c.x), x1 = x(c.y);
        if (VALUED) return fmaf(v.x, x0, v.y * x1);
        return x0 + x1;
    }
};
template <bool VALUED, bool SMEM>
struct Unit<1, VALUED, SMEM> {
    int32_t c; float v;
    __device__ __forceinline__ void load(const int32_t* col, const float* val, int s) {
        c = ld_i1<SMEM>(col + s);
        if (VALUED) v = ld_f1<SMEM>(val + s);
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
        epi.write(ent, -1, s);
    }
}

// The per-warp work of a workload is a flat sequence of "units" (one vector load per lane);
// each batch issues UB independent unit loads per lane (8 slots per lane in flight), then the
// gathers, then the sums; row boundaries fall at fixed unit counts (warp-uniform), where the
// row is reduced (row major: shuffles inside its lane group) and written.
//
// Row major (CSR-vector, L80-L82): lpr lanes per row (power of two covering w/4 int4 units,
// <= 32), rps = 32/lpr rows per step, upl = ceil(w/4/lpr) units per lane per row.
// wc / wv: the workload's first slot (global memory, or its copy in shared memory when SMEM).
template <bool VALUED, bool SMEM, class X, class Epi>
__device__ __forceinline__ void run_rm(const TileArgs& a, const WlDesc& d, const int32_t* wc,
                                       const float* wv, const X& x, Epi& epi, int lane) {
    constexpr int UB = X::kRmUnits;                      // int4 units per lane per batch
    const int w4 = d.w >> 2;                             // int4 groups per row
    const int lpr = w4 >= 32 ? 32 : (w4 <= 1 ? 1 : (1 << (32 - __clz(w4 - 1))));
    const int lg = __ffs(lpr) - 1;
    const int rps = 32 >> lg;
    const int sub = lane >> lg, sl = lane & (lpr - 1);
    const int upl = (w4 + lpr - 1) >> lg;                // units per lane per row
    const int steps = (d.h + rps - 1) / rps;
    const int V = steps * upl;                           // virtual units of this lane
    float acc = 0.0f;
    uint32_t ent_open = PAD_ROW;
    int32_t eix_open = -1;
    typename Epi::Pre pre_open{};
    Unit<4, VALUED, SMEM> u[UB];
    bool ok[UB];
    uint32_t ent_s[UB];
    int32_t eix_s[UB];
    // issue the slot loads (and row entries) of the batch starting at virtual unit b0
    auto issue = [&](int b0, Unit<4, VALUED, SMEM>* uu, bool* okk, uint32_t* en, int32_t* ei) {
        #pragma unroll
        for (int j = 0; j < UB; ++j) {
            const int v = b0 + j;
            const int step = v / upl, q = sl + (v - step * upl) * lpr;
            const int r = step * rps + sub;
            okk[j] = v < V && r < d.h && q < w4;
            if (okk[j]) uu[j].load(wc + r * d.w, VALUED ? wv + r * d.w : nullptr, 4 * q);
            // a row's entry and its epilogue operands are fetched when the row starts, so their
            // latency overlaps the row's slot loads and gathers
            // ei = -2 where no row starts: the entry-order epilogue state of a row is requested
            // with its row entry, without waiting for it (prefetch_rm)
            const bool starts = v < V && v % upl == 0 && sl == 0 && r < d.h;
            if constexpr (Epi::kEntryState) ei[j] = starts ? d.row_base + r : -2;
            else ei[j] = d.row_base + r;
            en[j] = starts ? __ldg(a.row_id + d.row_base + r) : PAD_ROW;
        }
    };
    issue(0, u, ok, ent_s, eix_s);
    for (int v0 = 0; v0 < V; v0 += UB) {
        typename Epi::Pre pre_s[UB];
        #pragma unroll
        for (int j = 0; j < UB; ++j) {
            if constexpr (Epi::kEntryState)
                pre_s[j] = (d.kind == KIND_SPLIT) ? typename Epi::Pre{} : epi.prefetch_rm(ent_s[j], eix_s[j], a.has_acc);
            else
                pre_s[j] = (d.kind == KIND_SPLIT) ? typename Epi::Pre{} : epi.prefetch(ent_s[j], eix_s[j]);
        }
        #pragma unroll
        for (int j = 0; j < UB; ++j) {
            const int v = v0 + j;
            if (v >= V) break;                           // warp-uniform
            if (v % upl == 0) { ent_open = ent_s[j]; eix_open = eix_s[j]; pre_open = pre_s[j]; }
            if (ok[j]) acc += u[j].dot(x);
            if ((v + 1) % upl == 0) {                    // row boundary (warp-uniform)
                for (int o = lpr >> 1; o >= 1; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
                if (ent_open != PAD_ROW) {
                    if (d.kind == KIND_SPLIT) finish_split(a, d, ent_open, acc, epi);
                    else epi.commit(ent_open, eix_open, acc, pre_open);
                }
                acc = 0.0f;
            }
        }
        issue(v0 + UB, u, ok, ent_s, eix_s);
    }
}

// Column major (ELL, L84): thread per row over 32-row slabs; the workload is a linear stream of
// 32*KV-slot units (unit u of lane l at slot u*32*KV + l*KV), a row ends every nk = w/KV units.
// The row entries (and partial y of accumulating rows) of every row ending in a batch are
// loaded with the batch.
template <int KV, bool VALUED, bool SMEM, class X, class Epi>
__device__ __forceinline__ void run_cm(const TileArgs& a, const WlDesc& d, const int32_t* wc,
                                       const float* wv, const X& x, Epi& epi, int lane) {
    constexpr int UB = ((VALUED ? X::kCmSlotsV : X::kCmSlotsP) + KV - 1) / KV;  // slots per lane in flight
    const int nk = d.w / KV;
    const int slabs = d.h >> 5;
    const int total = slabs * nk;
    const uint32_t* rid = a.row_id + d.row_base + lane;
    const int32_t* cb = wc + lane * KV;
    const float* vb = VALUED ? wv + lane * KV : nullptr;
    float acc = 0.0f;
    Unit<KV, VALUED, SMEM> u[UB];
    uint32_t ent[UB];
    auto issue = [&](int b0, Unit<KV, VALUED, SMEM>* uu, uint32_t* en) {
        #pragma unroll
        for (int j = 0; j < UB; ++j) {
            const int q = b0 + j;
            en[j] = PAD_ROW;
            if (q < total) {
                uu[j].load(cb, vb, q * (32 * KV));
                if ((q + 1) % nk == 0) en[j] = __ldg(rid + 32 * (q / nk));
            }
        }
    };
    issue(0, u, ent);
    for (int u0 = 0; u0 < total; u0 += UB) {
        typename Epi::Pre pre[UB];
        #pragma unroll
        for (int j = 0; j < UB; ++j) {
            if constexpr (Epi::kEntryState)
                pre[j] = epi.prefetch_rm(ent[j], (u0 + j + 1) % nk == 0 && u0 + j < total
                                                     ? d.row_base + lane + 32 * ((u0 + j) / nk) : -2, a.has_acc);
            else
                pre[j] = epi.prefetch(ent[j], d.row_base + lane + 32 * ((u0 + j) / nk));
        }
        #pragma unroll
        for (int j = 0; j < UB; ++j) {
            const int uu = u0 + j;
            if (uu >= total) break;                      // warp-uniform
            acc += u[j].dot(x);
            if ((uu + 1) % nk == 0) {                    // row end (warp-uniform)
                if (ent[j] != PAD_ROW) epi.commit(ent[j], d.row_base + lane + 32 * (uu / nk), acc, pre[j]);
                acc = 0.0f;
            }
        }
        issue(u0 + UB, u, ent);
    }
}

// TILE-COO workload (Observation 3): whole rows back to back, the last slot of each row
// flagged (COO_END).  The warp takes 32 slots per step, one per lane, and sums each row with a
// segmented inclusive scan over the lanes (Hillis-Steele with head flags: the paper's "binary
// reduction" that checks whether two operands belong to the same row, done with shuffles instead
// of serialised branches); the row open at the end of a step carries into the next.  Lanes that
// end a row write it (row index = rows ended before it in the workload).  Fixed order:
// deterministic.
template <bool VALUED, bool SMEM, class X, class Epi>
__device__ __forceinline__ void run_coo(const TileArgs& a, const WlDesc& d, const int32_t* wc,
                                        const float* wv, const X& x, Epi& epi, int lane) {
    float carry = 0.0f;                      // sum of the row open at the start of the step
    int32_t row = 0;                         // rows ended before this step
    for (int s0 = 0; s0 < d.w; s0 += 32) {
        const uint32_t cw = (uint32_t)(SMEM ? wc[s0 + lane] : __ldcs(wc + s0 + lane));
        const bool end = (cw & COO_END) != 0u;
        const int32_t c = (int32_t)(cw & ~COO_END);
        float v = x(c);                       // sentinel (padding) -> 0
        if (VALUED) v *= SMEM ? wv[s0 + lane] : __ldcs(wv + s0 + lane);
        const unsigned ends = __ballot_sync(0xffffffffu, end);
        // head of a segment: lane 0 or the lane after a row end
        bool head = lane == 0 || ((ends >> (lane - 1)) & 1u);
        #pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const float t = __shfl_up_sync(0xffffffffu, v, o);
            const bool th = __shfl_up_sync(0xffffffffu, head, o);
            if (lane >= o && !head) { v += t; head = th; }
        }
        // lanes of the step's first segment continue the row carried in
        const unsigned first_end = ends ? (unsigned)__ffs(ends) - 1u : 32u;
        if ((unsigned)lane <= first_end) v += carry;
        if (end) {
            const int32_t r = row + __popc(ends & ((1u << lane) - 1u));
            const uint32_t ent = __ldg(a.row_id + d.row_base + r);
            epi.write(ent, d.row_base + r, v);
        }
        // the open row's running sum (lane 31 when it does not end a row)
        const float last = __shfl_sync(0xffffffffu, v, 31);
        carry = (ends >> 31) & 1u ? 0.0f : last;
        row += __popc(ends);
    }
}

// zero-length rows (remainder tile): every row of every slab gets value 0
template <class Epi>
__device__ __forceinline__ void run_zero(const TileArgs& a, const WlDesc& d, Epi& epi, int lane) {
    for (int r0 = 0; r0 < d.h; r0 += 128) {
        uint32_t ent[4];
        #pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int r = r0 + 32 * j + lane;
            ent[j] = r < d.h ? __ldg(a.row_id + d.row_base + r) : PAD_ROW;
        }
        #pragma unroll
        for (int j = 0; j < 4; ++j)
            if (ent[j] != PAD_ROW) epi.write(ent[j], d.row_base + r0 + 32 * j + lane, 0.0f);
    }
}

template <bool VALUED, bool SMEM, class X, class Epi>
__device__ __forceinline__ void dispatch_cm(const TileArgs& a, const WlDesc& d, const int32_t* wc,
                                            const float* wv, const X& x, Epi& epi, int lane) {
    if (d.kvec == 4) run_cm<4, VALUED, SMEM>(a, d, wc, wv, x, epi, lane);
    else if (d.kvec == 2) run_cm<2, VALUED, SMEM>(a, d, wc, wv, x, epi, lane);
    else run_cm<1, VALUED, SMEM>(a, d, wc, wv, x, epi, lane);
}

__device__ __forceinline__ WlDesc load_desc(const WlDesc* p) {
    const int4* dp = reinterpret_cast<const int4*>(p);
    int4 d0 = __ldg(dp), d1 = __ldg(dp + 1);
    WlDesc d;
    d.off = (int64_t)(((uint64_t)(uint32_t)d0.y << 32) | (uint32_t)d0.x);
    d.row_base = d0.z; d.w = d0.w; d.h = d1.x;
    d.kind = (uint8_t)(d1.y & 0xff); d.kvec = (uint8_t)((d1.y >> 8) & 0xff);
    d.split_id = d1.z; d.chunk = d1.w;
    return d;
}

template <bool VALUED, bool SMEM, class X, class Epi>
__device__ __forceinline__ void run_workload(const TileArgs& a, const WlDesc& d, const int32_t* wc,
                                             const float* wv, const X& x, Epi& epi, int lane) {
    if (d.kind == KIND_COO) run_coo<VALUED, SMEM>(a, d, wc, wv, x, epi, lane);
    else if (d.kind != KIND_CM) run_rm<VALUED, SMEM>(a, d, wc, wv, x, epi, lane);
    else if (d.w == 0) run_zero(a, d, epi, lane);
    else dispatch_cm<VALUED, SMEM>(a, d, wc, wv, x, epi, lane);
}

constexpr int kPrefetchAhead = TC_PF_AHEAD;

template <bool VALUED>
__device__ __forceinline__ void prefetch_workload(const TileArgs& a, int64_t j) {
    const WlDesc d = load_desc(a.desc + j);
    const uint32_t bytes = (uint32_t)((int64_t)d.h * d.w * 4 + 15) & ~15u;
    if (bytes == 0) return;
    bulk_prefetch_l2(a.col + d.off, bytes);
    if (VALUED) bulk_prefetch_l2(a.val + d.off, bytes);
}

template <bool STAGED, bool VALUED, class Epi>
__global__ void __launch_bounds__(kThreads, STAGED ? 1 : TC_MINB) tc_spmv_tile(TileArgs a, Epi epi_in) {
    extern __shared__ float xs[];
    // programmatic dependent launch (standalone multi-launch products, "restart a
    // kernel for each tile"): the grid was launched while the previous launch (x relabel or tile)
    // finished its last workloads; wait for it to complete and flush.  A no-op for launches
    // without the PDL attribute (the solvers' graphs, single-launch plans).
    asm volatile("griddepcontrol.wait;" ::: "memory");
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
#if TC_X_POLICY
    x.pol = policy_evict_last();
#endif
    const int lane = threadIdx.x & 31;
    const int64_t gw = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
    const int64_t G = (int64_t)gridDim.x * kWarps;
#if TC_DYN
    // Hybrid schedule: all but the last two rounds of workloads are dealt round robin (warp gw
    // takes gw, gw + G, ...; their slots are bulk-prefetched into L2 two workloads ahead); the
    // last rounds are claimed from the launch's counter, so the launch ends within about one
    // workload of its last claim whatever the mix of workload costs.  The claim is issued a whole
    // workload before its result is needed.  The last warp out resets the counters for the next
    // launch on the stream.
    const int64_t n_wl = a.wl_end - a.wl_begin;
    const int64_t rounds = n_wl / G;
    // launches of fewer than eight rounds stay fully dealt (measured on c3 youtube: claiming
    // there costs more than the imbalance it removes)
    const int64_t s_end = rounds >= 8 && rounds > TC_DYN ? (rounds - TC_DYN) * G : n_wl;
    // the dealt sequence gw, gw + G, ... runs through the first dynamic round (s_end + gw)
    const int64_t dealt_end = s_end + G < n_wl ? s_end + G : n_wl;
    if (lane == 0) {
        for (int q = 0; q < kPrefetchAhead; ++q) {
            const int64_t jn = gw + q * G;
            if (jn < dealt_end) prefetch_workload<VALUED>(a, a.wl_begin + jn);
        }
    }
    for (int64_t j = gw; j < s_end; j += G) {
        const WlDesc d = load_desc(a.desc + a.wl_begin + j);
        const int64_t jn = j + (int64_t)kPrefetchAhead * G;
        if (kPrefetchAhead >= 0 && lane == 0 && jn < dealt_end) prefetch_workload<VALUED>(a, a.wl_begin + jn);
        run_workload<VALUED, false>(a, d, a.col + d.off, VALUED ? a.val + d.off : nullptr, x, epi, lane);
    }
    // dynamic rounds: the first workload is still dealt (no burst of claims at the boundary);
    // warps that finish early claim the rest
    // kDynQ queues (queue q holds s_end + G + q + kDynQ*i) spread the claims over as many
    // addresses: same-address atomics serialise at one L2 slice
    const int q = (int)(gw % kDynQ);
    int64_t jc = s_end + gw;
    while (jc < n_wl) {
        const WlDesc d = load_desc(a.desc + a.wl_begin + jc);
        if (kPrefetchAhead == 0 && lane == 0) prefetch_workload<VALUED>(a, a.wl_begin + jc);
        int64_t jf = 0;
        if (lane == 0) jf = s_end + G + q + (int64_t)kDynQ * atomicAdd(a.sched + q, 1u);   // used after the workload
        run_workload<VALUED, false>(a, d, a.col + d.off, VALUED ? a.val + d.off : nullptr, x, epi, lane);
        if (kPrefetchAhead > 0 && lane == 0 && jf < n_wl) prefetch_workload<VALUED>(a, a.wl_begin + jf);
        jc = __shfl_sync(0xffffffffu, jf, 0);
    }
    __syncwarp();                                         // converged warps at the block barrier
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(a.sched + kDynQ, 1u) == gridDim.x - 1u)
            for (int i = 0; i <= kDynQ; ++i) a.sched[i] = 0u;
    }
    (void)gw; (void)G;
#else
    // the warp's first workloads: prefetch their slots into L2 (bulk, asynchronous)
    if (lane == 0) {
        for (int q = 0; q < kPrefetchAhead; ++q) {
            const int64_t jn = a.wl_begin + gw + q * G;
            if (jn < a.wl_end) prefetch_workload<VALUED>(a, jn);
        }
    }
    for (int64_t j = a.wl_begin + gw; j < a.wl_end; j += G) {
        const WlDesc d = load_desc(a.desc + j);
        // keep kPrefetchAhead workloads of this warp in flight from HBM into L2
        const int64_t jn = j + (int64_t)kPrefetchAhead * G;
        if (kPrefetchAhead >= 0 && lane == 0 && jn < a.wl_end) prefetch_workload<VALUED>(a, jn);
        run_workload<VALUED, false>(a, d, a.col + d.off, VALUED ? a.val + d.off : nullptr, x, epi, lane);
    }
#endif
    // this CTA's workloads are done: the next launch may start (triggering at kernel start instead
    // measured slower on c2 multi-tile plans: profiles/r02_pdl.log)
    asm volatile("griddepcontrol.launch_dependents;");
    epi.end();
}

// Epilogue interface: prefetch(ent, e) loads what the row's write needs (the partial sum of
// earlier tiles when FLAG_ACC, epilogue operands) early; commit(ent, e, v, pre) stores the row's
// value or applies the fused epilogue; write(ent, e, v) = commit(ent, e, v, prefetch(ent, e)).
// prefetch_rm(ent, e, has_acc) is the one-pass tiles' form: e >= 0 is a row entry index whose
// entry-order state is loaded without consulting ent (its load may still be in flight), e = -1 a
// split row (state through fpos), e = -2 nothing; ent is read only for FLAG_ACC when has_acc.
// e is the index of the row entry in row_id[] (consecutive lanes -> consecutive entries, so
// per-row epilogue state kept in entry order is read and written coalesced); -1 for split rows.
// y = A x writer (no epilogue)
struct EpiStore {
    float* y;
    struct Pre { float acc; };
    __device__ __forceinline__ bool begin() { return true; }
    __device__ __forceinline__ void end() {}
    __device__ __forceinline__ Pre prefetch(uint32_t ent, int32_t) const {
        return Pre{(ent != PAD_ROW && (ent & FLAG_ACC)) ? y[ent & ROW_MASK] : 0.0f};
    }
    static constexpr bool kEntryState = true;    // one-pass tiles: prefetch_rm / prefetch_entry
    __device__ __forceinline__ Pre prefetch_rm(uint32_t ent, int32_t e, int32_t) const { return prefetch(ent, e); }
    __device__ __forceinline__ Pre prefetch_entry(int32_t) const { return Pre{0.0f}; }
    __device__ __forceinline__ void commit(uint32_t ent, int32_t, float v, const Pre& pre) { y[ent & ROW_MASK] = v + pre.acc; }
    __device__ __forceinline__ void write(uint32_t ent, int32_t e, float v) { commit(ent, e, v, prefetch(ent, e)); }
    // two-phase tiles: per-row state of entries [e0, e0 + n) into L2 ahead of the rows (none here)
    __device__ __forceinline__ void prefetch_rows(int64_t, int32_t, uint64_t) const {}
};

// A launch whose rows are all first touches (a plan's first tile): no accumulating rows, so the
// epilogue's prefetch needs only the entry-order state and never looks at the row entry, whose
// load may still be in flight (ncu source view: the FLAG_ACC test on it was the one-pass SpMV's
// top stall).  Same arithmetic and stores as Epi.
template <class Epi>
struct FirstTouch : Epi {
    static constexpr bool kEntryState = true;
    FirstTouch() = default;
    __host__ __device__ explicit FirstTouch(const Epi& e) : Epi(e) {}
    __device__ __forceinline__ typename Epi::Pre prefetch_rm(uint32_t, int32_t e, int32_t) const {
        return this->prefetch_entry(e);
    }
};

}  // namespace tc
