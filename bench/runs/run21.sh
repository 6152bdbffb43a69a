python -m pytest tests/test_gpu_dist.py -x -q 2>&1 | grep -vE "^\s+File|^    " | tail -4
export VARIANTS='[{"num_tiles":0,"workload_size":1024}]'
for pf in 0 8192 16384 24576; do echo "== prefix $pf"; TCSPMV_PREFIX=$pf python bench/explore_spmv.py c2 2>&1 | tail -1 | cut -c1-150; TCSPMV_PREFIX=$pf python bench/explore_spmv.py c2 --pattern 2>&1 | tail -1 | cut -c1-150; done
TCSPMV_PREFIX=16384 python bench/explore_pr.py c2 2>&1 | tail -3
