/* A plain C99 consumer of the C ABI (include/spmv.h): no Python, no torch.  Host-only calls only
 * (bitonic partition, a host-only plan, its layout decoded back to COO), so it runs without a GPU.
 * Prints "ok" on success; any mismatch exits non-zero with a message. */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "spmv.h"

static int fail(const char* what) {
    fprintf(stderr, "FAIL %s: %s\n", what, spmv_last_error());
    return 1;
}

int main(void) {
    /* S:L477 example: lengths [9,7,5,4,3,1], P = 2 -> {9,4,3} / {7,5,1} */
    const int64_t len[6] = {9, 7, 5, 4, 3, 1};
    int32_t owner[6];
    if (bitonic_partition(6, len, 2, owner) != SPMV_OK) return fail("bitonic_partition");
    const int32_t want[6] = {0, 1, 1, 0, 0, 1};
    for (int i = 0; i < 6; ++i)
        if (owner[i] != want[i]) { fprintf(stderr, "FAIL owner[%d] = %d\n", i, owner[i]); return 1; }
    /* a 4 x 5 matrix, host-only plan (device = -1), decoded back to COO */
    const int64_t rp[5] = {0, 3, 3, 5, 8};
    const int32_t col[8] = {0, 2, 4, 1, 2, 0, 3, 4};
    const float val[8] = {1, 2, 3, 4, 5, 6, 7, 8};
    spmv_options opt;
    spmv_options_default(&opt);
    opt.tile_width = 2;
    opt.num_tiles = 1;
    opt.workload_size = 4;
    spmv_plan plan = NULL;
    if (spmv_plan_create(4, 5, 8, rp, col, val, &opt, -1, &plan) != SPMV_OK) return fail("spmv_plan_create");
    spmv_plan_stats_t st;
    if (spmv_plan_stats(plan, &st) != SPMV_OK) return fail("spmv_plan_stats");
    if (st.n_rows != 4 || st.n_cols != 5 || st.nnz != 8 || st.num_tiles != 1) { fprintf(stderr, "FAIL stats\n"); return 1; }
    int32_t r[8], c[8];
    float v[8];
    if (spmv_plan_to_coo(plan, r, c, v) != SPMV_OK) return fail("spmv_plan_to_coo");
    /* every input entry appears exactly once (order is the layout's) */
    int seen[8] = {0};
    for (int k = 0; k < 8; ++k) {
        int hit = -1;
        for (int i = 0; i < 4 && hit < 0; ++i)
            for (int64_t e = rp[i]; e < rp[i + 1]; ++e)
                if (r[k] == i && c[k] == col[e] && v[k] == val[e] && !seen[e]) { hit = (int)e; break; }
        if (hit < 0) { fprintf(stderr, "FAIL coo entry %d (%d,%d,%g)\n", k, r[k], c[k], v[k]); return 1; }
        seen[hit] = 1;
    }
    /* errors come back as status codes with a message, never as aborts */
    if (spmv_execute(plan, NULL, NULL, NULL) == SPMV_OK) { fprintf(stderr, "FAIL execute(NULL)\n"); return 1; }
    if (spmv_plan_create(2, 2, 1, rp, col, val, NULL, -1, &plan) == SPMV_OK) { fprintf(stderr, "FAIL bad CSR accepted\n"); return 1; }
    spmv_plan_destroy(plan);
    printf("ok\n");
    return 0;
}
