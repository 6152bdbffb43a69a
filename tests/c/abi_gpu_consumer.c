/* A plain C99 consumer of the C ABI on the GPU (no Python, no torch, no CUDA runtime calls of its
 * own): reads a CSR matrix, x and a graph from binary files written by the test, runs
 * spmv_execute_host (host buffers; the library copies) and the one-shot pagerank(), and writes y
 * and p as float32 files for the test to compare against the fp64 oracle. */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "spmv.h"

static void* slurp(const char* path, size_t bytes) {
    FILE* f = fopen(path, "rb");
    if (!f) { fprintf(stderr, "cannot open %s\n", path); exit(2); }
    void* p = malloc(bytes ? bytes : 1);
    if (bytes && fread(p, 1, bytes, f) != bytes) { fprintf(stderr, "short read %s\n", path); exit(2); }
    fclose(f);
    return p;
}

static void spit(const char* path, const void* p, size_t bytes) {
    FILE* f = fopen(path, "wb");
    if (!f || fwrite(p, 1, bytes, f) != bytes) { fprintf(stderr, "cannot write %s\n", path); exit(2); }
    fclose(f);
}

int main(int argc, char** argv) {
    if (argc != 5) { fprintf(stderr, "usage: dir n m_spmv m_graph\n"); return 2; }
    const char* d = argv[1];
    const int64_t n = atoll(argv[2]), m = atoll(argv[3]), mg = atoll(argv[4]);
    char path[4096];
    snprintf(path, sizeof path, "%s/rp.bin", d);   int64_t* rp = slurp(path, (n + 1) * 8);
    snprintf(path, sizeof path, "%s/col.bin", d);  int32_t* col = slurp(path, m * 4);
    snprintf(path, sizeof path, "%s/val.bin", d);  float* val = slurp(path, m * 4);
    snprintf(path, sizeof path, "%s/x.bin", d);    float* x = slurp(path, n * 4);
    snprintf(path, sizeof path, "%s/grp.bin", d);  int64_t* grp = slurp(path, (n + 1) * 8);
    snprintf(path, sizeof path, "%s/gcol.bin", d); int32_t* gcol = slurp(path, mg * 4);
    spmv_plan plan = NULL;
    if (spmv_plan_create(n, n, m, rp, col, val, NULL, 0, &plan) != SPMV_OK) {
        fprintf(stderr, "plan: %s\n", spmv_last_error()); return 1;
    }
    float* y = malloc(n * 4);
    if (spmv_execute_host(plan, x, y, NULL) != SPMV_OK) { fprintf(stderr, "execute: %s\n", spmv_last_error()); return 1; }
    snprintf(path, sizeof path, "%s/y.bin", d); spit(path, y, n * 4);
    spmv_plan_destroy(plan);
    float* p = malloc(n * 4);
    spmv_iter_result res;
    if (pagerank(n, mg, grp, gcol, NULL, NULL, NULL, 0, p, &res) != SPMV_OK) {
        fprintf(stderr, "pagerank: %s\n", spmv_last_error()); return 1;
    }
    snprintf(path, sizeof path, "%s/p.bin", d); spit(path, p, n * 4);
    printf("%d\n", res.iterations);
    return 0;
}
