python -m pytest tests/test_gpu_spmv.py tests/test_gpu_iter.py -x -q 2>&1 | tail -4
export VARIANTS='[{"num_tiles":0,"workload_size":1024},{"num_tiles":0,"workload_size":512},{"tile_width":24576,"num_tiles":1,"workload_size":1024},{"tile_width":24576,"num_tiles":3,"workload_size":1024},{"tile_width":12288,"num_tiles":8,"workload_size":1024},{"tile_width":24576,"num_tiles":3,"workload_size":1024,"stage_x":0}]'
for v in default t1024 t256; do
  echo "=== $v"
  if [ $v = default ]; then L=$PWD/paper_1103_2405_b200/lib/libtcspmv.so; else L=$PWD/paper_1103_2405_b200/lib/libtcspmv_$v.so; fi
  TCSPMV_LIB=$L python bench/explore_spmv.py c2 2>&1 | tail -6 | cut -c1-140
  TCSPMV_LIB=$L python bench/explore_spmv.py c2 --pattern 2>&1 | tail -6 | cut -c1-140
done
