python -m pytest tests -m gpu -x -q 2>&1 | grep -vE "^\s+File|^    " | tail -6
export VARIANTS='[{"num_tiles":0,"workload_size":1024},{"num_tiles":0,"workload_size":512},{"tile_width":49152,"num_tiles":1,"workload_size":1024}]'
for v in default B2; do
  echo "=== $v"
  if [ $v = default ]; then L=$PWD/paper_1103_2405_b200/lib/libtcspmv.so; else L=$PWD/paper_1103_2405_b200/lib/libtcspmv_$v.so; fi
  TCSPMV_LIB=$L python bench/explore_spmv.py c2 2>&1 | tail -3 | cut -c1-120
  TCSPMV_LIB=$L python bench/explore_spmv.py c2 --pattern 2>&1 | tail -3 | cut -c1-120
  VARIANTS='[{"num_tiles":0,"workload_size":1024}]' TCSPMV_LIB=$L python bench/explore_pr.py c2
done
