// plan.h -- internal types of the tiled-composite plan (Format v1).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "spmv.h"

namespace tc {

constexpr uint32_t FLAG_ACC = 1u << 29;    // row already written by an earlier tile: y += v
constexpr uint32_t FLAG_FINAL = 1u << 30;  // no later tile touches the row: value is final
constexpr uint32_t ROW_MASK = (1u << 29) - 1;
constexpr uint32_t PAD_ROW = 0xFFFFFFFFu;  // padding row of a column-major slab
enum : uint8_t { KIND_RM = 0, KIND_CM = 1, KIND_SPLIT = 2, KIND_COO = 3 };
// TILE-COO workloads (orient = 3, dense tiles): whole rows back to back, the last slot of
// each row carries this flag in its column word
constexpr uint32_t COO_END = 1u << 31;

// One warp's workload (Solution 3): a w x h rectangle of slots.  32 bytes, read once per warp.
struct WlDesc {
    int64_t off;       // first slot
    int32_t row_base;  // first row entry in row_id[]
    int32_t w;         // RM / SPLIT: padded width (multiple of align_rm); CM: width (row length)
    int32_t h;         // RM: rows; CM: slab rows (multiple of ell_h); SPLIT: 1
    uint8_t kind;
    uint8_t kvec;      // CM: 4/2/1 consecutive slots per lane (k-interleave); RM: 4
    uint16_t pad_;
    int32_t split_id;  // SPLIT: index into the split table, else -1
    int32_t chunk;     // SPLIT: chunk index
};
static_assert(sizeof(WlDesc) == 32, "descriptor must be 32 bytes");

struct TileInfo {
    int64_t col_lo = 0, col_hi = 0;     // relabelled column range [lo, hi)
    int64_t wl_begin = 0, wl_end = 0;   // workload range
    int64_t nnz = 0, rows = 0, slots = 0;
    int32_t wl = 0;                     // workload size WL used for this tile
    int32_t threshold = 0;              // composite threshold: first CM row length (0 = none)
    int32_t staged = 0;                 // x segment staged in shared memory
    double pred_us = 0.0;               // performance-model estimate
};

// Relabelled copy of the input (steps a1/a2): per row, entries ordered by relabelled column.
struct Prepared {
    int64_t n_rows = 0, n_cols = 0, nnz = 0;
    bool pattern = false;
    std::vector<int32_t> perm;        // relabelled position -> original column
    std::vector<int32_t> inv;         // original column -> relabelled position
    std::vector<int64_t> collen;      // column length by relabelled position (non-increasing)
    std::vector<int64_t> rp;          // row pointer (copy of the input)
    std::vector<int32_t> kcol;        // relabelled column per entry, ascending within a row
    std::vector<float> kval;          // values in the same order (empty for pattern)
    int64_t max_row_len = 0;
};

struct HostLayout {
    std::vector<TileInfo> tiles;      // num_tiles dense tiles + 1 remainder
    std::vector<WlDesc> desc;
    std::vector<uint32_t> row_id;
    std::vector<int32_t> slot_col;
    std::vector<float> slot_val;
    std::vector<int32_t> split;       // 3 per split row: row entry, n_chunks, partial_base
    int64_t n_chunks = 0;
    // host view arrays (filled on demand)
    std::vector<int64_t> v_tiles, v_off;
    std::vector<int32_t> v_row_base, v_w, v_h, v_split_id, v_chunk;
    std::vector<uint8_t> v_kind, v_kvec;
};

struct BuildParams {
    int32_t tile_width = 1;
    int32_t num_tiles = 0;
    std::vector<int32_t> wl;          // num_tiles + 1 values
    int32_t align_rm = 8;
    bool split = true;
    bool camping = false;
    int32_t ell_h = 32;
    int32_t orient = 0;               // 0 composite, 1 row major only, 2 column major only,
                                      // 3 TILE-COO (dense tiles COO, remainder composite)
};

// Alg. 3's orientation rule (row major iff w >= h), or a forced single format (f2 ablations).
inline bool row_major(int32_t orient, int64_t w, int64_t hq) {
    return orient == 1 ? w > 0 : (orient == 2 ? false : w >= hq);
}

// errors are reported through set_error() + status
void set_error(const std::string& msg);

spmv_status prepare(int64_t n_rows, int64_t n_cols, int64_t nnz, const int64_t* row_ptr,
                    const int32_t* col, const float* val, bool pattern, Prepared& P, bool keep_order = false);
int32_t paper_tile_count(const Prepared& P, int64_t tile_width);
// Sorted (descending) in-tile row-length histogram of every tile for a given tiling:
// hist[t] = vector of (length, count) pairs, lengths descending; zero rows go to the remainder.
void tile_histograms(const Prepared& P, int64_t tile_width, int32_t num_tiles,
                     std::vector<std::vector<std::pair<int64_t, int64_t>>>& hist);
void tile_histograms_multi(const Prepared& P, int64_t tile_width, const std::vector<int32_t>& num_tiles,
                           std::vector<std::vector<std::vector<std::pair<int64_t, int64_t>>>>& out);
spmv_status pack_layout(const Prepared& P, const BuildParams& bp, HostLayout& L);

}  // namespace tc
