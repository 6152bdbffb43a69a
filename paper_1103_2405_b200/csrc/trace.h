// trace.h -- NVTX phase ranges (SURVEY.md 5 "Tracing and profiling"): plan build (prepare, tune,
// pack, upload), SpMV launches, solver runs, the row-partitioned exchange.  Header-only NVTX 3:
// free when no tool is attached; ncu / nsys show the ranges.
#pragma once
#include <nvtx3/nvToolsExt.h>

namespace tc {
struct Range {
    explicit Range(const char* name) { nvtxRangePushA(name); }
    ~Range() { nvtxRangePop(); }
    Range(const Range&) = delete;
    Range& operator=(const Range&) = delete;
};
}  // namespace tc
