/*
 * spmv.h -- C ABI of the B200-native tiled-composite SpMV library (libtcspmv.so).
 *
 * Method: Yang, Parthasarathy & Sadayappan, "Fast Sparse Matrix-Vector Multiplication on GPUs:
 * Implications for Graph Mining", PVLDB 4(4), 2011 (cited as PAPER.md Lnn = line of the text).
 *
 * The library computes y = A x for an n_rows x n_cols sparse matrix A in CSR (PAPER.md L291,
 * App. B problem statement) through the paper's TILE-COMPOSITE representation:
 *   - columns reordered by decreasing length (Solution 2, L66),
 *   - the dense leading columns cut into fixed-width tiles whose x segment stays on chip
 *     (Solution 1, L56-L60; Alg. 1), the rest one composite remainder tile (L90-L92),
 *   - inside each tile, rows ranked by length and packed into ~WL-entry workloads, each a w x h
 *     rectangle run by one warp: row major / CSR-vector when w >= h, column major / ELL otherwise
 *     (Solution 3, L88, L94),
 * and the power iterations PageRank (Eq. 6), HITS (Eq. 8) and Random Walk with
 * Restart (Eq. 9) on top of it, on one B200 or row-partitioned over several (Sec. 3.2).
 *
 * Conventions for every function:
 *   - returns spmv_status; SPMV_OK = 0.  Nothing throws or aborts across this boundary; the
 *     message of the last non-OK status of the calling thread is spmv_last_error().
 *   - host input arrays are borrowed for the duration of the call and copied; the caller keeps
 *     ownership.  "_dev" pointers are device pointers owned by the caller (e.g. torch tensors).
 *   - streams are cudaStream_t passed as void* (NULL = legacy default stream).
 *   - indices: row_ptr int64 (nnz may exceed 2^31), column ids int32, n_rows < 2^29.
 *   - there is no CPU fallback: without a CUDA device every device entry point returns
 *     SPMV_ECUDA.
 */
#ifndef TCSPMV_H
#define TCSPMV_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    SPMV_OK = 0,
    SPMV_EINVAL = 1,      /* null pointer, negative size, row_ptr not monotone, column out of range,
                             bad option value */
    SPMV_EDIM = 2,        /* inconsistent dimensions */
    SPMV_ENOTSQUARE = 3,  /* graph algorithm given a non-square matrix */
    SPMV_ERANGE = 4,      /* query >= n, P > rows, n_rows >= 2^29, too many tiles */
    SPMV_EROWSPLIT = 5,   /* split_long_rows = 0 and a workload size is below the tile's longest row */
    SPMV_ETABLE = 6,      /* performance table missing or malformed */
    SPMV_ENOMEM = 7,      /* host or device allocation failed */
    SPMV_ECUDA = 8,       /* CUDA runtime error, or no device */
    SPMV_ENCCL = 9,       /* NCCL error */
    SPMV_ENOCONV = 10     /* max_iter reached before tol; outputs are still written */
} spmv_status;

typedef struct spmv_plan_s* spmv_plan;
typedef struct spmv_comm_s* spmv_comm;
typedef struct spmv_solver_s* spmv_solver;

/* Options of the format builder (Sec. 3.1) and of the auto-tuner (Sec. 3.3).
 * spmv_options_default() fills: tile_width 0 (auto), num_tiles -1 (auto), workload_size -1
 * (auto), workload_sizes NULL, align_rm 8, split_long_rows 1, camping_pad 0, pattern 0,
 * ell_h 32, stage_x 1, perf_table_path NULL, orient 0, two_phase -1, pb_region / pb_chunk /
 * pb_xcap / pb_group 0 (defaults), keep_col_order 0. */
typedef struct {
    int32_t tile_width;      /* columns per dense tile (paper: 64K, L60); 0 = chosen by the tuner */
    int32_t num_tiles;       /* dense tiles before the remainder; -1 = auto (Alg. 1 + B200 model);
                                0 = single composite tile (the whole matrix is the remainder) */
    int32_t workload_size;   /* WL for every tile; -1 = auto per tile (Alg. 2) */
    const int32_t* workload_sizes; /* optional, num_tiles + 1 explicit WLs (last = remainder) */
    int32_t align_rm;        /* row-major width alignment in slots (paper: warp size 32, L88;
                                B200 default 8 = one 32-byte sector); multiple of 4 on device */
    int32_t split_long_rows; /* 1: rows longer than WL become one-row chunks combined in chunk
                                order (B200; reading R21).  0: paper lower bound WL >= longest row */
    int32_t camping_pad;     /* 1: +64 slots after workloads of 512k slots (L96); default 0 */
    int32_t pattern;         /* 1: values implicitly 1.0 (val may be NULL) */
    int32_t ell_h;           /* column-major slab height (warp size); must be 32 to execute */
    int32_t stage_x;         /* 1: dense tiles stage their x segment in shared memory */
    const char* perf_table_path; /* JSON offline table (Sec. 3.3); NULL = built-in B200 table */
    int32_t orient;          /* workload orientation (§8(f) f2 ablations; the model covers the
                                single-format cases): 0 = composite (Alg. 3: row major iff
                                w >= h), 1 = row major only (CSR-vector), 2 = column major only (ELL),
                                -1 = the one the performance model predicts fastest.
                                Rows of length 0 and split chunks are unaffected. */
    int32_t two_phase;       /* execution of the tiles: -1 = chosen by the performance
                                model (default), 0 = one-pass tiles (x gathered through L1/L2),
                                1 = two-phase tiles: every column tile's x segment is staged in
                                shared memory (Solution 1, L56-L60) and its products are written
                                to per-row-bin regions, which a second phase sums row by row with
                                the composite split (Solution 3, L88) */
    int32_t pb_region;       /* two-phase: products per row-bin region (0 = 8192; 32..65535) */
    int32_t pb_chunk;        /* two-phase: entries per column chunk (0 = 8192) */
    int32_t pb_xcap;         /* two-phase: columns per chunk x segment (0 = 6144, or 4096 when
                              * 6144 would not leave two CTAs per SM; <= 65536) */
    int64_t pb_group;        /* two-phase: products per group of bins kept L2-resident between the
                                phases (0 = chosen from the L2 size) */
    int32_t keep_col_order;  /* 1: skip the column relabel (Solution 2) and keep the caller's
                                column order -- for an x laid out by someone else (the row-
                                partitioned solvers read the exchange buffer directly); no dense
                                tiles then (Alg. 1 needs length-sorted columns), only L2-sized ones
                                when x exceeds L2.  One-pass tiles only.  Default 0. */
} spmv_options;

void spmv_options_default(spmv_options* opt);

/* Summary of a built plan. */
typedef struct {
    int64_t n_rows, n_cols, nnz;
    int32_t num_tiles;          /* dense tiles (the remainder tile is extra) */
    int32_t tile_width;
    int64_t n_workloads, n_slots, n_row_entries, n_split, n_chunks;
    int64_t device_bytes;       /* device memory held by the plan */
    double predicted_us;        /* performance-model estimate of one spmv_execute (Eq. 2) */
    double build_ms;            /* host build time */
    int32_t wl[64];             /* per tile WL (tile i < num_tiles; [num_tiles] = remainder) */
    int64_t tile_nnz[64];
    int64_t tile_rows[64];      /* rows touched per tile */
    int64_t tile_col_lo[64], tile_col_hi[64];
    int32_t tile_staged[64];
    double tile_predicted_us[64];
    int32_t composite_threshold[64]; /* first row length stored column major in each tile */
    int32_t resident_warps;     /* warps of one persistent tile launch (MAX_ACT_WARP of Eq. 1) */
    int32_t perf_table_loaded;  /* 1: measured offline table (Sec. 3.3), 0: built-in estimate */
    int32_t two_phase;          /* 1: the plan executes as two-phase tiles (spmv_options.two_phase) */
    int32_t pb_groups;          /* two-phase: groups, chunks, bins, long-row bins */
    int64_t pb_chunks, pb_bins, pb_long_bins;
    double one_pass_predicted_us;  /* model estimate of the one-pass tiles (Alg. 3 / Eq. 2) */
    double two_phase_predicted_us; /* model estimate of the two-phase tiles */
    int32_t orient;             /* workload orientation in use (0 composite, 1 row major, 2 column
                                   major; with spmv_options.orient = -1 the model's choice) */
} spmv_plan_stats_t;

/* Host view of the layout arrays (Format v1), valid while the plan lives, when the
 * plan keeps its host copy (host-only plans always do).  All pointers are plan-owned. */
typedef struct {
    int64_t n_cols, n_workloads, n_row_entries, n_slots, n_split, n_tiles_total;
    const int32_t* perm;        /* [n_cols] relabelled position -> original column */
    const int64_t* tiles;       /* [n_tiles_total][4] col_lo, col_hi, wl_begin, wl_end */
    const int64_t* desc_off;    /* per workload: first slot */
    const int32_t* desc_row_base, *desc_w, *desc_h, *desc_split_id, *desc_chunk;
    const uint8_t* desc_kind, *desc_kvec;
    const uint32_t* row_id;     /* row | 1<<29 (accumulate) | 1<<30 (final); 0xFFFFFFFF = pad */
    const int32_t* slot_col;    /* tile-relative column; sentinel = tile width */
    const float* slot_val;      /* NULL for pattern plans */
    const int32_t* split;       /* [n_split][3] row entry, n_chunks, partial_base */
} spmv_layout_view;

/* Build the tiled-composite plan of A (host CSR, copied) and upload it to `device`.
 * device = -1 builds a host-only plan (layout inspection / export; cannot execute).
 * val may be NULL when opt->pattern = 1.  Errors: EINVAL, EDIM, ERANGE, EROWSPLIT, ENOMEM, ECUDA. */
spmv_status spmv_plan_create(int64_t n_rows, int64_t n_cols, int64_t nnz, const int64_t* row_ptr,
                             const int32_t* col_idx, const float* val, const spmv_options* opt,
                             int device, spmv_plan* out);
void spmv_plan_destroy(spmv_plan plan);

/* y = A x.  x_dev: n_cols floats in the caller's column order; y_dev: n_rows floats in the
 * caller's row order.  Asynchronous on `stream`.  Deterministic: bitwise identical across runs.
 * The plan's device scratch serves one product at a time: a call on a different stream than the
 * plan's previous product first waits (cudaStreamWaitEvent) for that product, so products of one
 * plan never overlap; use one plan per stream for concurrent products. */
spmv_status spmv_execute(spmv_plan plan, const float* x_dev, float* y_dev, void* stream);

/* Same product with x already in relabelled column order (xp_dev[k] = x[perm[k]]), as the
 * power iterations keep it; skips the x permutation kernel. */
spmv_status spmv_execute_permuted(spmv_plan plan, const float* xp_dev, float* y_dev, void* stream);

/* spmv_execute with a CUDA event between launches; synchronises and writes the device time of
 * every launch (x permutation first, then each tile) to launch_ms[0 .. spmv_plan_launches()).
 * For measurement (bench.py's roofline of the dominant kernel). */
spmv_status spmv_execute_timed(spmv_plan plan, const float* x_dev, float* y_dev, void* stream,
                               float* launch_ms, int32_t max_launches);

/* Host -> device -> host convenience: copies x (host), executes, copies y back, synchronises. */
spmv_status spmv_execute_host(spmv_plan plan, const float* x_host, float* y_host, void* stream);

/* Pipelined host -> device -> host over `count` independent products: y_b = A x_b for
 * b = 0 .. count-1, x_host row-major [count][n_cols], y_host row-major [count][n_rows] (both
 * caller-owned; pinned memory lets the copies run asynchronously). Three plan-owned device buffer
 * pairs and two plan-owned copy streams overlap the H2D copy of x_{b+1}, the product b on
 * `stream` and the D2H copy of y_{b-1}; every product still copies its own x in and its own y
 * out. Synchronises before returning. Same per-product operation as spmv_execute (PAPER.md
 * L291). Errors: SPMV_EINVAL (null pointer, count < 0), SPMV_ECUDA. */
spmv_status spmv_execute_host_batch(spmv_plan plan, const float* x_host, float* y_host,
                                    int32_t count, void* stream);

spmv_status spmv_plan_stats(spmv_plan plan, spmv_plan_stats_t* out);
spmv_status spmv_plan_layout(spmv_plan plan, spmv_layout_view* out);
/* Write the layout arrays (Format v1) to `path` for the bit-exact format oracle
 * (oracle/format_ref.py).  File: 8-byte magic "TCSPMV1\0", then int64
 * n_rows, n_cols, n_workloads, n_row_entries, n_slots, n_split, n_tiles_total, valued (0/1),
 * then, little endian and back to back: perm i32[n_cols], tiles i64[n_tiles_total*4],
 * desc_off i64[nw], desc_row_base/w/h/split_id/chunk i32[nw] each, desc_kind u8[nw],
 * desc_kvec u8[nw], row_id u32[n_row_entries], slot_col i32[n_slots], slot_val f32[n_slots]
 * (valued plans only), split i32[n_split*3].  Errors: EINVAL (null), ENOMEM (file not writable),
 * ECUDA (layout download). */
spmv_status spmv_plan_export(spmv_plan plan, const char* path);
/* Read a file written by spmv_plan_export back into a plan and upload it to `device` (-1: host
 * only) -- a checkpoint of the preprocessing (sort, tiling, packing: paid once per matrix, L98).
 * The tiling, WLs and layout are the file's; per-tile predictions are not stored (0).  Two-phase
 * plans have no Format v1 file.  Errors: EINVAL (unreadable / not Format v1 / truncated), ENOMEM,
 * ECUDA. */
spmv_status spmv_plan_import(const char* path, int device, spmv_plan* out);
/* Decode the layout back to COO (original row / column ids), padding dropped; arrays of nnz. */
spmv_status spmv_plan_to_coo(spmv_plan plan, int32_t* rows, int32_t* cols, float* vals);
/* Diagnostic (two-phase plans): one product with a per-item timeline.  trace_host receives
 * n_items x {SM id, start ns, reduce ready ns (0 for chunks), end ns} in work-queue order
 * (globaltimer).  Synchronises.  Errors: EINVAL (not a device two-phase plan, buffer too small). */
spmv_status spmv_pb_trace(spmv_plan plan, const float* x_dev, float* y_dev, void* stream,
                          int64_t* trace_host, int64_t n_items);
/* Number of kernel launches one spmv_execute issues (x permutation included). */
int32_t spmv_plan_launches(spmv_plan plan);

/* ---------------------------------------------------------------- power iterations (App. F) */
enum { SPMV_ALGO_PAGERANK = 0, SPMV_ALGO_HITS = 1, SPMV_ALGO_RWR = 2 };

typedef struct {
    double c;              /* PageRank damping (0.85, L430) / RWR c (0.9, L456); unused by HITS */
    double tol;            /* L1 stopping threshold on the change (reading R2); default 1e-6 */
    int32_t max_iter;      /* default 1000 */
    int32_t hits_norm;     /* 1 = halves sum to 1 (paper, L440; default), 2 = unit L2 halves */
    int32_t fixed_iters;   /* > 0: run exactly this many iterations (parity at equal k) */
    int32_t exchange;      /* multi-GPU only: 0 = one allgather of every non-empty column (default);
                            * 1 = needed columns: each rank receives only the values its rows read,
                            *     by grouped NCCL send/recv (spmv_needed_lists) */
    int32_t host_loop;     /* single GPU: 0 = the iterations run as a CUDA graph with a device-side
                            * WHILE loop (default); 1 = the host enqueues them in batches of 8 and
                            * reads the device's stop flag (same kernels and results; for profilers
                            * and sanitizers, which do not see inside conditional graph nodes) */
} spmv_iter_opts;
void spmv_iter_opts_default(spmv_iter_opts* o, int algo);

typedef struct {
    int32_t iterations;
    int32_t converged;
    double residual;       /* last L1 change */
    double ms_total;       /* device time of the iteration loop (CUDA events) */
    double us_per_iter;
    double predicted_us_per_iter;
    double phase_us[3];    /* row-partitioned solvers: mean per iteration of the local SpMV (with
                            * its fused epilogue), the exchange, and the rest (partial sums, HITS
                            * normalisation), from CUDA events between the phases; single GPU:
                            * {us_per_iter, 0, 0} */
} spmv_iter_result;

/* Graph input for all three: adjacency A of G = (V,E), CSR with row u listing the targets v of
 * u -> v (A(u,v) = 1, L414); duplicates collapse, self loops are kept.
 * A solver builds its plan once (preprocessing amortised over iterations, L98) and can run many
 * times; `comm` = NULL runs on one GPU, else the row-partitioned multi-GPU path (Sec. 3.2):
 * every rank passes the whole graph, owns the rows bitonic_partition gives it, runs its local
 * tiled-composite SpMV with the fused epilogue, and the next x plus the fp64 partials are
 * exchanged by one NCCL allgather per iteration.  HITS exchanges the raw product with its half
 * sums and normalises after the exchange; its stop decision lags one SpMV (the converged iterate
 * is the one returned). */
spmv_status spmv_solver_create(int algo, int64_t n, int64_t m, const int64_t* row_ptr,
                               const int32_t* col, const spmv_iter_opts* it,
                               const spmv_options* opt, spmv_comm comm, int device,
                               spmv_solver* out);
/* Row-partitioned solver from this rank's rows only (SURVEY 8(b) "*_local", for graphs too large
 * to hold whole on every rank): the caller owns the vertices owned_ids[0 .. n_local) (every vertex
 * of [0, n_global) owned by exactly one rank) and passes their rows of the iteration matrix with
 * global column ids -- PageRank: the in-neighbours u of each owned v (edges u -> v, Eq. 6;
 * duplicates already merged) plus out_degree[r] of each owned vertex; RWR: the neighbours in
 * A u A^T (Eq. 9; reading R8), out_degree NULL (the row length is the degree); HITS: rows
 * of the block matrix [[0, A^T], [A, 0]] (Eq. 8), owned_ids in [0, 2 n_global) -- row
 * v < n_global lists n_global + u for every edge u -> v, row n_global + u lists v -- and
 * out_degree NULL (a block row's length is also its column's length).  Ownership
 * and degrees of all vertices are exchanged once over the communicator (O(n) per rank); the
 * iteration is the allgather path of spmv_solver_create with comm.  Results and runs as for
 * spmv_solver_create (spmv_solver_result writes all n_global values on every rank).
 * On the loopback transport the ranks' builds run one at a time (they share the host's memory).
 * Errors: EINVAL (null pointer, PageRank without out_degree, HITS with out_degree, overlapping /
 * missing ownership, exchange = 1), ERANGE (id outside [0, n_global), HITS [0, 2 n_global)),
 * ENCCL, ECUDA. */
spmv_status spmv_solver_create_local(int algo, int64_t n_global, int64_t n_local, const int32_t* owned_ids,
                                     const int64_t* row_ptr, const int32_t* col, const int32_t* out_degree,
                                     const spmv_iter_opts* it, const spmv_options* opt, spmv_comm comm,
                                     int device, spmv_solver* out);
/* Run the power iteration from the initial vector (RWR: query node `query`).  Synchronises. */
spmv_status spmv_solver_run(spmv_solver s, int64_t query, void* stream, spmv_iter_result* res);
/* Copy the result to host, in the caller's vertex order: PageRank p [n], RWR r [n],
 * HITS authority a [n] in out0 and hub h [n] in out1. */
spmv_status spmv_solver_result(spmv_solver s, float* out0, float* out1);
spmv_status spmv_solver_plan_stats(spmv_solver s, spmv_plan_stats_t* out);
/* Change the stopping rule between runs (spmv_iter_opts tol, max_iter, fixed_iters; reading R2):
 * the plan, the exchange layout and every other option stay, so one build serves runs to several
 * iteration counts (preprocessing amortised, L98).  Errors: EINVAL (null, tol < 0, max_iter < 1,
 * fixed_iters < 0). */
spmv_status spmv_solver_set_stop(spmv_solver s, double tol, int32_t max_iter, int32_t fixed_iters);
int32_t spmv_solver_launches_per_iter(spmv_solver s);
void spmv_solver_destroy(spmv_solver s);

/* Batched RWR (the paper's 25 random queries, L448): the Q <= 32 queries of an
 * RWR solver iterate together as one SpMM over the same layout (lanes = queries: one 128-byte x
 * row per stored entry instead of Q random gathers).  The loop runs until every query's L1 change
 * is below tol (or fixed_iters); res->residual is the largest.  Synchronises.
 * Errors: EINVAL (not an RWR solver, multi-GPU solver, Q outside [1, 32]), ERANGE (query). */
spmv_status spmv_solver_run_batch(spmv_solver s, const int64_t* queries, int32_t Q, void* stream,
                                  spmv_iter_result* res);
/* The batched results, query-major: out[q * n + u] = r_q(u), caller order. */
spmv_status spmv_solver_result_batch(spmv_solver s, float* out);

/* One-shot wrappers: create, run, copy result, destroy. */
spmv_status pagerank(int64_t n, int64_t m, const int64_t* row_ptr, const int32_t* col,
                     const spmv_iter_opts* it, const spmv_options* opt, spmv_comm comm,
                     int device, float* p_out, spmv_iter_result* res);
spmv_status hits(int64_t n, int64_t m, const int64_t* row_ptr, const int32_t* col,
                 const spmv_iter_opts* it, const spmv_options* opt, spmv_comm comm,
                 int device, float* auth_out, float* hub_out, spmv_iter_result* res);
spmv_status rwr(int64_t n, int64_t m, const int64_t* row_ptr, const int32_t* col, int64_t query,
                const spmv_iter_opts* it, const spmv_options* opt, spmv_comm comm,
                int device, float* r_out, spmv_iter_result* res);

/* ---------------------------------------------------------------- multi-GPU (Sec. 3.2) */
/* Bitonic (snake) partition of rows by length over P ranks (L108, reading R25):
 * owner_out[i] in [0,P).  Row counts differ by at most 1.  Errors: EINVAL, ERANGE (P > rows). */
spmv_status bitonic_partition(int64_t n_rows, const int64_t* row_len, int32_t P, int32_t* owner_out);

/* Ownership and slot layout of the row-partitioned path: owner_out[i] = bitonic owner of row i,
 * local_index_out[i] = its position among its owner's rows (ascending row id), *slot_rows = the
 * largest per-rank row count (every rank's allgather slot holds that many values).
 * Errors as bitonic_partition. */
spmv_status spmv_partition_plan(int64_t n_rows, const int64_t* row_len, int32_t P, int32_t* owner_out,
                                int64_t* local_index_out, int64_t* slot_rows);

/* Needed-columns exchange lists for the row partition `owner` (the paper's row
 * partition, Sec. 3.2, exchanging only what each partition reads, L106-L108).  M is the
 * n x n iteration matrix (CSR: row i reads the columns col[row_ptr[i] .. row_ptr[i+1])).  For rank
 * `rank`: send_count[q] = number of vertices owned by `rank` that rows owned by q read, recv_count[q]
 * = number of vertices owned by q that rows owned by `rank` read (both 0 for q = rank); send_ids /
 * recv_ids (optional, sized by the sums) receive the lists concatenated in rank order, each list
 * ascending by vertex id -- the order both ends of a message use.  Host only (no device needed).
 * Errors: EINVAL (null pointer, P < 1, rank outside [0,P), column outside [0,n)), ERANGE (owner
 * outside [0,P)), ENOMEM. */
spmv_status spmv_needed_lists(int64_t n, const int64_t* row_ptr, const int32_t* col, const int32_t* owner,
                              int32_t P, int32_t rank, int64_t* send_count, int64_t* recv_count,
                              int32_t* send_ids, int32_t* recv_ids);

/* Communicator over NCCL (loaded at run time).  nccl_unique_id: the 128-byte ncclUniqueId,
 * created by rank 0 with spmv_comm_unique_id() and broadcast by the caller (e.g. over a torch
 * process group).  world = 1 is valid (no NCCL calls). */
spmv_status spmv_comm_unique_id(void* id_out_128_bytes);
spmv_status spmv_comm_create(int rank, int world, const void* nccl_unique_id, int device,
                             spmv_comm* out);
/* Test transport: `world` logical ranks in one process on one `device`, written
 * to out[0 .. world).  Each handle is driven by its own host thread (one rank each, as with NCCL);
 * the per-iteration exchange, the needed-columns segments and the metadata allgather become
 * device-to-device copies between the ranks' buffers behind the same interface, ordered by
 * events and host barriers.  Lets the row-partitioned code path (slots, offsets, packing, rank-
 * order partial sums) run and be checked on one GPU.  Destroy every handle.  Errors: EINVAL, ECUDA. */
spmv_status spmv_comm_create_loopback(int world, int device, spmv_comm* out);
/* Row slices of one solver on one device (for matrices whose plan cannot be built in one piece on
 * the host, e.g. BASELINE configs[4]'s 11 G-entry HITS block): as spmv_comm_create_loopback, but
 * the ranks' solvers share one double-buffered exchange buffer (allocated by rank 0's solver at
 * its first run): each rank writes its own slot, and the per-iteration exchange is only the
 * ordering -- every rank's stream waits for every other rank's slot -- with no copies.  Same
 * results as the loopback transport, bit for bit.  spmv_iter_opts.exchange must be 0.
 * Errors: EINVAL, ECUDA; at the first run ENOMEM if the shared buffer cannot be allocated. */
spmv_status spmv_comm_create_slices(int world, int device, spmv_comm* out);
void spmv_comm_destroy(spmv_comm comm);

const char* spmv_last_error(void);
const char* spmv_version(void);

#ifdef __cplusplus
}
#endif
#endif /* TCSPMV_H */
