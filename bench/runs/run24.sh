export VARIANTS='[{"num_tiles":0,"workload_size":1024}]'
for co in -1 0 10 25; do echo "== carveout $co"; TCSPMV_CARVEOUT=$co python bench/explore_spmv.py c2 2>&1 | tail -1 | cut -c1-120; TCSPMV_CARVEOUT=$co python bench/explore_spmv.py c2 --pattern 2>&1 | tail -1 | cut -c1-120; done
