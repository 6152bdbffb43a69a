python -m pytest tests/test_gpu_dist.py -x -q 2>&1 | grep -vE "^\s+File|^    " | tail -25
export VARIANTS='[{"num_tiles":0,"workload_size":512},{"num_tiles":0,"workload_size":1024},{"num_tiles":0,"workload_size":2048},{"tile_width":49152,"num_tiles":2,"workload_size":1024}]'
for v in default B C D; do
  echo "=== $v"
  if [ $v = default ]; then L=$PWD/paper_1103_2405_b200/lib/libtcspmv.so; else L=$PWD/paper_1103_2405_b200/lib/libtcspmv_$v.so; fi
  TCSPMV_LIB=$L python bench/explore_spmv.py c2 2>&1 | tail -4 | cut -c1-120
  TCSPMV_LIB=$L python bench/explore_spmv.py c2 --pattern 2>&1 | tail -4 | cut -c1-120
done
export VARIANTS='[{"num_tiles":0,"workload_size":1024}]'
python bench/explore_pr.py c2
