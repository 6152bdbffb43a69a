// pb_kernels.cuh -- sm_100a kernel of the two-phase tiles (pb.h).
//
// One persistent launch, warp-specialised: in every CTA one producer warp claims work items from a
// device counter in queue order E(0) E(1) R(0) E(2) R(1) ... (expand chunks of group g, reduce bins
// of group g) and moves each item's streams into a shared-memory stage with 1-D bulk copies (TMA,
// cp.async.bulk, SASS UBLKCP), kPbStages items ahead of the consumer warps, which compute out of
// shared memory only:
//   expand: buf[gbase + k + run[r]] = a * x[c]  (column/run words, values, x segment and run table
//           all staged; entries in (bin, column, row) order, so a warp's 32 consecutive entries
//           store into one or two contiguous runs: whole-line writes), products stored with an L2
//           evict-last policy -- the group's regions stay in L2 until its reduces read them.
//   reduce: the producer first waits (acquire on the group counter) until every chunk of the group
//           has finished, then stages the bin's region, position block, row order and row meta;
//           the consumers discard the region's lines from L2 (dead: no write-back), and sum every
//           row in a fixed order -- warp per row at or above the composite threshold (positions
//           contiguous, lane-strided, shuffle tree), thread per row below it (32-row column-major
//           slabs) -- handing the value to the epilogue (Epi::commit) exactly as the one-pass tile
//           kernel's final row write does.  A PB_LONG bin (one row longer than a region) is summed
//           by the consumers straight from L2 (fixed strided order + fixed tree).
// Deterministic: every row is summed in an order fixed by the layout; no atomics on values.
// No deadlock: claims are in queue order, a reduce depends only on earlier items, so the earliest
// unfinished item can always proceed.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "pb.h"
#include "plan.h"
#include "tc_async.cuh"

namespace tc {

#ifndef PB_CWARPS
#define PB_CWARPS 8
#endif
constexpr int kPbConsumerWarps = PB_CWARPS;
constexpr int kPbConsumers = 32 * kPbConsumerWarps;
constexpr int kPbThreads = kPbConsumers + 32;          // + the producer warp
constexpr int kPbWarps = kPbThreads / 32;
#ifndef PB_STATIC
#define PB_STATIC 1
#endif
#ifndef PB_STAGES
#define PB_STAGES 2
#endif
constexpr int kPbStages = PB_STAGES;

struct PbArgs {
    const PbItem* items;         // work queue (descriptors in queue order)
    const int32_t* runs;         // padded by 4
    const uint32_t* cd;          // padded by 4
    const float* val;            // padded by 4; nullptr: pattern
    const uint16_t* pos;
    const uint32_t* prow;        // padded by 4
    const uint32_t* pmeta;       // padded by 4
    const int32_t* group_chunks;
    int32_t n_items, n_groups;
    float* buf;
    const float* x;              // input vector (16-byte aligned), the plan's column order
    int64_t n_cols;
    int32_t stage_bytes;         // per stage, header included
    uint32_t* ctl;               // [0] queue head, [1] CTAs finished, [2 + g] chunks done in group g
    int64_t* trace;              // diagnostic (spmv_pb_trace): per item {sm, start, ready, end} ns
};

// stage header, written by the producer before it arrives on the stage's full barrier
struct PbStage {
    PbItem d;                    // the item (kind kPbEnd: no more items)
    int32_t item;                // queue position (trace)
    int32_t o_a, o_b, o_c, o_d;  // byte offsets of the staged streams
    //   expand: column/run words, values, x segment, run table
    //   reduce: region, positions, row order, row meta
    int32_t pre_a, pre_b, pre_c; // elements before the first one (16-byte alignment)
    int64_t t_ready;             // trace: the reduce's dependency satisfied
};
static_assert(sizeof(PbStage) <= 128, "stage header fits 128 bytes");
constexpr int32_t kPbEnd = -1;

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_release_add(uint32_t* p, uint32_t v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_keep(float* p, float v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void discard_l2_line(const void* p) {
    asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void consumer_sync() {    // named barrier 1: the consumer warps only
    asm volatile("bar.sync 1, %0;" ::"n"(kPbConsumers) : "memory");
}
__device__ __forceinline__ int64_t gtimer() {
    int64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ uint32_t smid() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
    return r;
}
__device__ __forceinline__ PbItem load_item(const PbItem* p) {
    const int4* q = reinterpret_cast<const int4*>(p);
    int4 a = __ldg(q), b = __ldg(q + 1), c = __ldg(q + 2);
    PbItem r;
    r.a0 = (int64_t)(((uint64_t)(uint32_t)a.y << 32) | (uint32_t)a.x);
    r.a1 = (int64_t)(((uint64_t)(uint32_t)a.w << 32) | (uint32_t)a.z);
    r.a2 = (int64_t)(((uint64_t)(uint32_t)b.y << 32) | (uint32_t)b.x);
    r.n = b.z; r.b0 = b.w; r.b1 = c.x; r.b2 = c.y; r.group = c.z; r.kind = c.w;
    return r;
}

// broadcast a plain struct from lane `src` (word by word)
template <class T>
__device__ __forceinline__ T shfl_pod(const T& v, int src) {
    static_assert(sizeof(T) % 4 == 0, "shuffled structs are whole 32-bit words");
    T out;
    const uint32_t* a = reinterpret_cast<const uint32_t*>(&v);
    uint32_t* b = reinterpret_cast<uint32_t*>(&out);
    #pragma unroll
    for (int i = 0; i < (int)(sizeof(T) / 4); ++i) b[i] = __shfl_sync(0xffffffffu, a[i], src);
    return out;
}

// ------------------------------------------------------------------ producer (one thread)
__device__ __forceinline__ void stage_copy(uint8_t* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                           uint64_t pol) {
    if (bytes) bulk_g2s(dst, src, bytes, bar, pol);
}

template <bool VALUED, class Epi>
__device__ __forceinline__ void produce(const PbArgs& a, int32_t it, const PbItem& t, uint8_t* stage,
                                        uint64_t* full, uint64_t pol_stream, uint64_t pol_x, const Epi& epi) {
    PbStage* h = reinterpret_cast<PbStage*>(stage);
    uint8_t* d = stage + 128;
    h->item = it;
    h->t_ready = 0;
    h->d = t;
    if (it >= a.n_items) {
        h->d.kind = kPbEnd;
        mbar_arrive(full);
        return;
    }
    uint32_t off = 0;
    if (t.kind == PB_ITEM_EXPAND) {
        const int64_t e0 = t.a0, run0 = t.a2;
        const int32_t col0 = t.b0, span = t.b1, nrun = t.b2;
        const int64_t e_al = e0 & ~3LL;
        const uint32_t be = (uint32_t)(((e0 & 3) + t.n + 3) & ~3) * 4u;
        const int64_t x_al = col0 & ~3LL;
        const int32_t pre_x = (int32_t)(col0 - x_al);
        // the x copy stops at the last whole 16-byte group inside [0, n_cols); the (< 4) floats
        // after it are stored by this thread before it arrives
        const int64_t x_end = x_al + ((pre_x + span + 3) & ~3);
        const int64_t x_bulk_end = x_end <= a.n_cols ? x_end : (a.n_cols & ~3LL);
        const int64_t r_al = run0 & ~3LL;
        const uint32_t br = (uint32_t)(((run0 & 3) + nrun + 3) & ~3) * 4u;
        h->pre_a = (int32_t)(e0 & 3); h->pre_b = pre_x; h->pre_c = (int32_t)(run0 & 3);
        h->o_a = 0; off = be;
        h->o_b = (int32_t)off; if (VALUED) off += be;
        h->o_c = (int32_t)off; off += (uint32_t)(x_end - x_al) * 4u;
        h->o_d = (int32_t)off;
        float* xs = reinterpret_cast<float*>(d + h->o_c);
        for (int64_t j = x_bulk_end; j < x_end && j < a.n_cols; ++j) xs[j - x_al] = __ldg(a.x + j);
        const uint32_t bx = (uint32_t)(x_bulk_end - x_al) * 4u;
        mbar_arrive_expect_tx(full, be * (VALUED ? 2u : 1u) + bx + br);
        stage_copy(d, a.cd + e_al, be, full, pol_stream);
        if (VALUED) stage_copy(d + h->o_b, a.val + e_al, be, full, pol_stream);
        stage_copy(d + h->o_c, a.x + x_al, bx, full, pol_x);
        stage_copy(d + h->o_d, a.runs + r_al, br, full, pol_stream);
    } else {
        {   // dependency: every chunk of the bin's group has stored its products
            const uint32_t need = (uint32_t)__ldg(a.group_chunks + t.group);
            while (ld_acquire(a.ctl + 2 + t.group) < need) __nanosleep(32);
            fence_proxy_async_global();          // the bulk copies below read those products
            if (a.trace) h->t_ready = gtimer();
        }
        const int64_t roff = t.a0, poff = t.a1, row0 = t.a2;
        const int32_t rlen = t.n, plen = t.b0, nrows = t.b1;
        const int64_t row_al = row0 & ~3LL;
        const uint32_t brow = (uint32_t)(((row0 & 3) + nrows + 3) & ~3) * 4u;
        h->pre_a = (int32_t)(row0 & 3);
        const bool lng = t.kind == PB_ITEM_LONG;
        const uint32_t breg = lng ? 0u : (uint32_t)((rlen + 3) & ~3) * 4u;
        const uint32_t bpos = lng ? 0u : (uint32_t)plen * 2u;
        h->o_a = 0; off = breg;
        h->o_b = (int32_t)off; off += bpos;
        h->o_c = (int32_t)off; off += brow;
        h->o_d = (int32_t)off;
        epi.prefetch_rows(row0, nrows, pol_stream);   // per-row epilogue state into L2
        mbar_arrive_expect_tx(full, breg + bpos + 2 * brow);
        stage_copy(d, a.buf + roff, breg, full, pol_stream);
        stage_copy(d + h->o_b, a.pos + poff, bpos, full, pol_stream);
        stage_copy(d + h->o_c, a.prow + row_al, brow, full, pol_stream);
        stage_copy(d + h->o_d, a.pmeta + row_al, brow, full, pol_stream);
    }
}

// ------------------------------------------------------------------ consumers (8 warps)
#ifndef PB_EXPAND_UNROLL
#define PB_EXPAND_UNROLL 4
#endif

template <bool VALUED>
__device__ __forceinline__ void consume_expand(const PbArgs& a, const PbStage& h, const uint8_t* d, int tid) {
    const uint32_t* cd = reinterpret_cast<const uint32_t*>(d + h.o_a) + h.pre_a;
    const float* vv = reinterpret_cast<const float*>(d + h.o_b) + h.pre_a;
    const float* xs = reinterpret_cast<const float*>(d + h.o_c) + h.pre_b;
    const int32_t* rt = reinterpret_cast<const int32_t*>(d + h.o_d) + h.pre_c;
    const int32_t n = h.d.n;
    float* dst = a.buf + h.d.a1;
    const uint64_t pol = policy_evict_last();
    constexpr int U = PB_EXPAND_UNROLL;
    for (int k0 = tid; k0 < n; k0 += kPbConsumers * U) {
        #pragma unroll
        for (int j = 0; j < U; ++j) {
            const int k = k0 + j * kPbConsumers;
            if (k < n) {
                const uint32_t w = cd[k];
#ifdef PB_EXP_NOXGATHER
                const float xv = xs[k & 1023];   // experiment: conflict-free x reads
#else
                const float xv = xs[w & 0xffffu];
#endif
#ifdef PB_EXP_COALESCED
                st_keep(a.buf + h.d.a0 + k + (rt[w >> 16] & 0), VALUED ? vv[k] * xv : xv, pol);   // experiment
#else
                st_keep(dst + k + rt[w >> 16], VALUED ? vv[k] * xv : xv, pol);
#endif
            }
        }
    }
    // the producer releases the chunk (group counter) once every consumer warp has arrived
}

template <class Epi>
__device__ __forceinline__ void consume_reduce(const PbArgs& a, const PbStage& h, const uint8_t* d, Epi& epi,
                                               int tid) {
    const int lane = tid & 31, warp = tid >> 5;
    const int64_t row0 = h.d.a2;
    const int32_t rlen = h.d.n, nrows = h.d.b1, nheavy = h.d.b2;
    const uint32_t* prow = reinterpret_cast<const uint32_t*>(d + h.o_c) + h.pre_a;
    const uint32_t* pmeta = reinterpret_cast<const uint32_t*>(d + h.o_d) + h.pre_a;
    const float* reg_g = a.buf + h.d.a0;
    const int nlines = (rlen + 31) >> 5;
    if (h.d.kind == PB_ITEM_LONG) {
        __shared__ float wsum[kPbConsumerWarps];
        float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
        int k = tid;
        for (; k + 3 * kPbConsumers < rlen; k += 4 * kPbConsumers) {
            #pragma unroll
            for (int j = 0; j < 4; ++j) acc[j] += __ldcg(reg_g + k + j * kPbConsumers);
        }
        for (; k < rlen; k += kPbConsumers) acc[0] += __ldcg(reg_g + k);
        float s = (acc[0] + acc[1]) + (acc[2] + acc[3]);
        for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) wsum[warp] = s;
        consumer_sync();
        for (int i = tid; i < nlines; i += kPbConsumers) discard_l2_line(reg_g + 32 * i);   // consumed
        if (tid == 0) {
            float t = 0.0f;
            for (int w = 0; w < kPbConsumerWarps; ++w) t += wsum[w];
            epi.write(prow[0], (int32_t)row0, t);
        }
        consumer_sync();
        return;
    }
    // the region lives in shared memory now: its lines are dead in L2 (no write-back)
    for (int i = tid; i < nlines; i += kPbConsumers) discard_l2_line(reg_g + 32 * i);
    const float* reg = reinterpret_cast<const float*>(d + h.o_a);
    const uint16_t* ps = reinterpret_cast<const uint16_t*>(d + h.o_b);
    // heavy rows: warp per row (CSR-vector).  The epilogue operands of the warp's next
    // 32 heavy rows are requested at once, one row per lane, and handed to lane 0 by shuffles.
    for (int r0 = warp; r0 < nheavy; r0 += 32 * kPbConsumerWarps) {
        const int rl = r0 + lane * kPbConsumerWarps;
        const uint32_t ent_l = rl < nheavy ? prow[rl] : PAD_ROW;
#ifdef PB_EXP_NOPRE
        const typename Epi::Pre pre_l{};
#else
        const typename Epi::Pre pre_l = epi.prefetch(ent_l, (int32_t)(row0 + rl));
#endif
        for (int j = 0; j < 32; ++j) {
            const int r = r0 + j * kPbConsumerWarps;
            if (r >= nheavy) break;
            const uint32_t m = pmeta[r];
            const int po = (int)(m & 0xffffu), ln = (int)(m >> 16);
            float acc = 0.0f;
            for (int k = lane; k < ln; k += 32) acc += reg[ps[po + k]];
            for (int o = 16; o >= 1; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            const typename Epi::Pre pre = shfl_pod(pre_l, j);
            if (lane == 0) epi.commit(prow[r], (int32_t)(row0 + r), acc, pre);
        }
    }
    // light rows: thread per row over column-major 32-row slabs (ELL); the epilogue
    // operands of all of a thread's rows are requested before any of them is summed
    constexpr int LR = 4;
    const int nlight = nrows - nheavy;
    for (int l0 = tid; l0 < nlight; l0 += LR * kPbConsumers) {
        uint32_t ent[LR], m[LR];
        typename Epi::Pre pre[LR];
        #pragma unroll
        for (int j = 0; j < LR; ++j) {
            const int li = l0 + j * kPbConsumers;
            const int r = nheavy + li;
            ent[j] = li < nlight ? prow[r] : PAD_ROW;
            m[j] = li < nlight ? pmeta[r] : 0u;
#ifdef PB_EXP_NOPRE
            pre[j] = typename Epi::Pre{};
#else
            pre[j] = epi.prefetch(ent[j], (int32_t)(row0 + r));
#endif
        }
        #pragma unroll
        for (int j = 0; j < LR; ++j) {
            const int li = l0 + j * kPbConsumers;
            if (li >= nlight) break;
            const int po = (int)(m[j] & 0xffffu), ln = (int)(m[j] >> 16);
            float acc = 0.0f;
            int k = 0;
            for (; k + 4 <= ln; k += 4) {
                const float v0 = reg[ps[po + 32 * k]], v1 = reg[ps[po + 32 * (k + 1)]];
                const float v2 = reg[ps[po + 32 * (k + 2)]], v3 = reg[ps[po + 32 * (k + 3)]];
                acc += v0; acc += v1; acc += v2; acc += v3;
            }
            for (; k < ln; ++k) acc += reg[ps[po + 32 * k]];
            epi.commit(ent[j], (int32_t)(row0 + nheavy + li), acc, pre[j]);
        }
    }
}

template <bool VALUED, class Epi>
__global__ void __launch_bounds__(kPbThreads) pb_spmv(PbArgs a, Epi epi_in) {
    extern __shared__ __align__(128) uint8_t pb_sm[];
    __shared__ __align__(8) uint64_t full[kPbStages], empty[kPbStages];
    Epi epi = epi_in;
    if (!epi.begin()) return;                              // iteration loop already converged
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kPbStages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], kPbConsumerWarps); }
        fence_barrier_init();
    }
    __syncthreads();
    if (warp == kPbConsumerWarps) {
        // ---- producer warp (lane 0 issues).  The next item is claimed while the current one is
        // issued and its descriptor loaded while the stage drains; claims stay in queue order.
        if (lane == 0) {
            const uint64_t pol_stream = policy_evict_first();
            const uint64_t pol_x = policy_evict_last();
            // stage s holds iteration pend_k[s]; pend_g[s] >= 0: an expand of that group whose
            // release (group counter) is due once the consumers have drained the stage.  The
            // consumers' stores are ordered before the release by the stage's empty barrier.
            int32_t pend_k[kPbStages], pend_g[kPbStages];
            for (int s = 0; s < kPbStages; ++s) { pend_k[s] = -1; pend_g[s] = -1; }
            auto retire = [&](int s) {
                if (pend_k[s] < 0) return;
                mbar_wait(&empty[s], (uint32_t)(pend_k[s] / kPbStages) & 1u);
                if (pend_g[s] >= 0) red_release_add(a.ctl + 2 + pend_g[s], 1u);
                pend_k[s] = -1; pend_g[s] = -1;
            };
#if PB_STATIC
            // static round robin: this CTA's items are blockIdx.x + k * gridDim.x (queue order), so
            // the next descriptor loads while the current item is issued (the grid is co-resident:
            // cooperative launch)
            int32_t it = (int32_t)blockIdx.x;
#else
            int32_t it = (int32_t)atomicAdd(a.ctl, 1u);
#endif
            PbItem t = it < a.n_items ? load_item(a.items + it) : PbItem{};
            for (int k = 0;; ++k) {
                const int s = k % kPbStages;
#if PB_STATIC
                const int32_t it_next = it < a.n_items ? it + (int32_t)gridDim.x : it;
                PbItem t_next = it_next < a.n_items ? load_item(a.items + it_next) : PbItem{};
#else
                const int32_t it_next = it < a.n_items ? (int32_t)atomicAdd(a.ctl, 1u) : it;
#endif
                retire(s);
                // a reduce may wait for expands of its group held by this CTA: release them first
                if (it < a.n_items && t.kind != PB_ITEM_EXPAND)
                    for (int q = 0; q < kPbStages; ++q)
                        if (pend_g[q] >= 0 && pend_g[q] <= t.group) retire(q);
                uint8_t* stage = pb_sm + (size_t)s * a.stage_bytes;
                if (a.trace && it < a.n_items) a.trace[4 * (int64_t)it + 1] = gtimer();
                produce<VALUED>(a, it, t, stage, &full[s], pol_stream, pol_x, epi);
                if (it >= a.n_items) break;
                pend_k[s] = k;
                pend_g[s] = t.kind == PB_ITEM_EXPAND ? t.group : -1;
                it = it_next;
#if PB_STATIC
                t = t_next;
#else
                if (it < a.n_items) t = load_item(a.items + it);
#endif
            }
            for (int q = 0; q < kPbStages; ++q) retire(q);
        }
        __syncwarp();
    } else {
        // ---- consumer warps
        const int tid = threadIdx.x;
        for (int k = 0;; ++k) {
            const int s = k % kPbStages;
            mbar_wait(&full[s], (uint32_t)(k / kPbStages) & 1u);
            const uint8_t* stage = pb_sm + (size_t)s * a.stage_bytes;
            const PbStage h = *reinterpret_cast<const PbStage*>(stage);
            if (h.d.kind == kPbEnd) break;
#if defined(PB_DRY)
            // experiment: data movement only (products and sums not computed)
#elif defined(PB_DRY_EXPAND)
            if (h.d.kind != PB_ITEM_EXPAND) consume_reduce(a, h, stage + 128, epi, tid);
#elif defined(PB_DRY_REDUCE)
            if (h.d.kind == PB_ITEM_EXPAND) consume_expand<VALUED>(a, h, stage + 128, tid);
#else
            if (h.d.kind == PB_ITEM_EXPAND) consume_expand<VALUED>(a, h, stage + 128, tid);
            else consume_reduce(a, h, stage + 128, epi, tid);
#endif
            __syncwarp();
            if (a.trace && tid == 0) {
                int64_t* r = a.trace + 4 * (int64_t)h.item;
                r[0] = smid(); r[2] = h.t_ready; r[3] = gtimer();
            }
            if (lane == 0) mbar_arrive(&empty[s]);
        }
    }
    epi.end();
    // the last CTA out resets the queue for the next launch on the stream
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(a.ctl + 1, 1u) == gridDim.x - 1u) {
            a.ctl[0] = 0u;
            for (int g = 0; g < a.n_groups; ++g) a.ctl[2 + g] = 0u;
            __threadfence();
            a.ctl[1] = 0u;
        }
    }
}

}  // namespace tc
