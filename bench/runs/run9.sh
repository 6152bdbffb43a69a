export VARIANTS='[{"num_tiles":0,"workload_size":1024},{"num_tiles":0,"workload_size":256},{"tile_width":24576,"num_tiles":1,"workload_size":1024},{"tile_width":24576,"num_tiles":3,"workload_size":1024},{"tile_width":12288,"num_tiles":8,"workload_size":1024},{"tile_width":24576,"num_tiles":3,"workload_size":1024,"stage_x":0}]'
for v in lean512x3 lean256x8 u768; do
  echo "=== $v"
  TCSPMV_LIB=$PWD/paper_1103_2405_b200/lib/libtcspmv_$v.so python bench/explore_spmv.py c2 2>&1 | tail -6 | cut -c1-140
  TCSPMV_LIB=$PWD/paper_1103_2405_b200/lib/libtcspmv_$v.so python bench/explore_spmv.py c2 --pattern 2>&1 | tail -6 | cut -c1-140
done
