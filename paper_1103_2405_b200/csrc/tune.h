// tune.h -- parameter choice (Sec. 3.3): tile width, tile count (Alg. 1), workload size per
// tile (Alg. 2) and the performance model PM(T, WL) (Alg. 3, Eq. 1-5).
#pragma once
#include <vector>

#include "plan.h"

struct spmv_plan_s;

namespace tc {

spmv_status choose_params(const Prepared& P, const spmv_options& opt, int sm_count,
                          BuildParams& bp, std::vector<double>& pred_us, int32_t* table_loaded = nullptr);
void predict_plan(spmv_plan_s& p, const std::vector<double>& pred_us);

}  // namespace tc
