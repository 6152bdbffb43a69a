// tune.h -- parameter choice (Sec. 3.3): tile width, tile count (Alg. 1), workload size per
// tile (Alg. 2) and the performance model PM(T, WL) (Alg. 3, Eq. 1-5).
#pragma once
#include <vector>

#include "pb.h"
#include "plan.h"

struct spmv_plan_s;

namespace tc {

spmv_status choose_params(const Prepared& P, const spmv_options& opt, int sm_count,
                          BuildParams& bp, std::vector<double>& pred_us, int32_t* table_loaded = nullptr);
void predict_plan(spmv_plan_s& p, const std::vector<double>& pred_us);
// two-phase tiles (pb.h): parameters from the options and the L2 budget, and the byte model
PbParams pb_params(const spmv_options& opt, int64_t n_cols, int64_t nnz);
double pb_predict_us(const spmv_options& opt, int64_t n_rows, int64_t n_cols, int64_t nnz, bool valued,
                     const PbParams& prm);
double pb_predict_items_us(const spmv_options& opt, int64_t items, bool valued);
// a streaming pass over `bytes` (one launch at the table's staging bandwidth): the HITS solvers'
// normalisation pass beside the modelled SpMV (the paper's "two vector division", L440)
double stream_pass_us(const spmv_options& opt, double bytes);

}  // namespace tc
