// pb.h -- two-phase tiles: the tiled-composite product with the x gathers taken off the L1/L2
// request path.
//
// Solution 1 of the paper keeps a tile's segment of x on chip so that the random
// reads of x are served from fast memory.  On B200 a random 4-byte gather that misses L1 costs one
// L2 sector request whatever its byte count, and the mid-degree columns of a power-law graph are
// touched less than once per SM per product, so no per-SM cache captures them.
// Two-phase tiles take the tiling to its limit: every column tile ("chunk", at most `xcap`
// columns) has its x segment staged in shared memory, and instead of accumulating into y (one
// random read-modify-write per entry) each entry's product a_ij * x_j is written to the row's
// slot in a per-row-bin region of a partial buffer.  A second phase sums every row of a bin out of
// its region, staged in shared memory, with the paper's composite split (Solution 3, L88, L94):
// rows at or above the threshold one warp per row (CSR-vector), shorter rows one thread per row
// over 32-row column-major slabs (ELL).  Both phases read and write HBM/L2 in whole lines; every
// random access is a shared-memory access.
//
//   expand (chunk c of group g): stage x[col0, col0 + span) and c's run table in shared memory;
//       for its entries (ordered by (bin, column, row)): buf[gbase + k + run[r(k)]] = a_k * x[col_k]
//   reduce (bin b of group g, after every chunk of g):  stage region b and its position block;
//       y[row] = sum_t region[pos[row][t]]   (fixed order: deterministic)
//
// Rows are grouped into bins (consecutive rows, region <= `rcap` products) and bins into groups
// (region sum <= `gcap`, so the live part of the partial buffer stays in L2); one persistent launch
// runs the work queue E(0) E(1) R(0) E(2) R(1) ... : a reduce item waits (device-side counter) for
// its group's expands, which were claimed before it.
#pragma once
#include <cstdint>
#include <vector>

namespace tc {

struct PbChunk {            // 48 B
    int64_t e0;             // first entry (cd / val index)
    int64_t gbase;          // buffer offset of the chunk's group
    int64_t run0;           // first run-table entry
    int32_t n;              // entries
    int32_t col0;           // first column of the x segment
    int32_t span;           // x segment length (<= xcap)
    int32_t nrun;           // runs (distinct bins) in the chunk
    int32_t group;
    int32_t pad_;
};
static_assert(sizeof(PbChunk) == 48, "PbChunk is 48 bytes");

enum : int32_t { PB_BIN = 0, PB_LONG = 1 };

struct PbBin {              // 48 B
    int64_t roff;           // region offset in the partial buffer (multiple of 32: whole lines)
    int64_t poff;           // position block offset in pos[] (multiple of 8)
    int64_t row0;           // first row of the bin in the two-phase row order
    int32_t rlen;           // products in the region
    int32_t plen;           // position block length (multiple of 8)
    int32_t nrows;
    int32_t nheavy;         // rows at or above the composite threshold (warp per row), first
    int32_t group;
    int32_t kind;           // PB_BIN, or PB_LONG: one row longer than rcap (streamed, no positions)
};
static_assert(sizeof(PbBin) == 48, "PbBin is 48 bytes");

// One work item of the device queue (queue order E(0) E(1) R(0) ...), the chunk or bin descriptor
// itself so that a claim is followed by a single 48-byte load.
enum : int32_t { PB_ITEM_EXPAND = 0, PB_ITEM_BIN = 1, PB_ITEM_LONG = 2 };
struct PbItem {             // 48 B
    int64_t a0;             // expand: e0      reduce: roff
    int64_t a1;             // expand: gbase   reduce: poff
    int64_t a2;             // expand: run0    reduce: row0
    int32_t n;              // expand: n       reduce: rlen
    int32_t b0;             // expand: col0    reduce: plen
    int32_t b1;             // expand: span    reduce: nrows
    int32_t b2;             // expand: nrun    reduce: nheavy
    int32_t group;
    int32_t kind;           // PB_ITEM_*
};
static_assert(sizeof(PbItem) == 48, "PbItem is 48 bytes");

struct PbParams {
    int32_t rcap = 6144;        // products per bin region (shared memory of one reduce)
    int32_t pcap = 9216;        // positions per bin block (<= 65535)
    int32_t maxrows = 1024;     // rows per bin (row order and meta staged with the region)
    int32_t xcap = 6144;        // columns per chunk x segment (shared memory of one expand); a
                                // layout whose stages would not fit two CTAs per SM is rebuilt
                                // with kPbXcapFallback (pb_build_fit)
    int32_t ccap = 4096;        // entries per chunk
    int32_t nrcap = 1024;       // runs per chunk (run table in shared memory)
    int32_t heavy = 32;         // composite threshold of the reduce: rows >= heavy are warp-per-row
    int64_t gcap = 6 << 20;     // products per group (live partial buffer kept in L2)
};

struct PbLayout {
    int64_t n_rows = 0, n_cols = 0, nnz = 0;
    bool pattern = false;
    PbParams prm;
    std::vector<PbChunk> chunks;
    std::vector<PbBin> bins;
    std::vector<int32_t> runs;          // per run: buffer offset (group-relative) - run start (chunk-local)
    std::vector<uint32_t> cd;           // per entry: (column - col0) | run index << 16
    std::vector<float> val;             // per entry (valued plans)
    std::vector<uint16_t> pos;          // per bin block: region-relative positions
    std::vector<uint32_t> prow;         // two-phase row order: row | FLAG_FINAL
    std::vector<uint32_t> pmeta;        // per row: position offset in its bin block | length << 16
    std::vector<int32_t> items;         // work queue: chunk c >= 0, bin b as ~b
    std::vector<int32_t> group_chunks;  // chunks per group
    int64_t buf_floats = 0;             // partial buffer length
    int32_t n_groups = 0;
    int64_t stage_bytes = 0;            // pb_stage_bytes
};

// Build the two-phase layout of an n_rows x n_cols CSR matrix (original row and column ids).
// Returns false (with set_error) when a parameter cannot hold the matrix.
bool pb_build(int64_t n_rows, int64_t n_cols, const int64_t* rp, const int32_t* col, const float* val,
              bool pattern, const PbParams& prm, PbLayout& L);

// Shared memory of one CTA's stages that still lets two CTAs share an SM (228 KB per SM, 1 KB
// reserved per CTA, the kernel's static shared memory): the persistent kernel needs two CTAs per SM
// to overlap its pipelines (one CTA per SM measured 1.47x slower on c2, profiles/r02_pb_xcap.log)
constexpr int64_t kPbTwoCtaSmem = 112 * 1024;   // two stages (kPbStages) per CTA
constexpr int32_t kPbXcapFallback = 4096;
// pb_build, and when the default x segment cap makes the stages too large for two CTAs per SM and
// the caller did not fix the cap, again with kPbXcapFallback
bool pb_build_fit(int64_t n_rows, int64_t n_cols, const int64_t* rp, const int32_t* col, const float* val,
                  bool pattern, PbParams prm, bool xcap_fixed, PbLayout& L);

// Bytes of one pipeline stage of the persistent CTA (pb_kernels.cuh): a 128-byte header plus the
// largest item's staged streams (expand: column/run words, values, x segment, run table; reduce:
// region, positions, row order, row meta), each from its 16-byte boundary.
int64_t pb_stage_bytes(const PbLayout& L);

}  // namespace tc
