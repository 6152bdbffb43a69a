# first-touch launches (plan's first tile) with an epilogue that never looks at the row entry vs prev
for r in 1 2; do
for L in libtcspmv_prev.so libtcspmv.so; do
  echo "lib $L"
  TCSPMV_LIB=$PWD/paper_1103_2405_b200/lib/$L VARIANTS='[{}]' timeout 600 python bench/explore_solver_plan.py c2 2>&1 | grep -v batch_fuse
  TCSPMV_LIB=$PWD/paper_1103_2405_b200/lib/$L timeout 600 python bench/explore_pb.py c2 '[{"two_phase":0},{"two_phase":0,"num_tiles":2,"tile_width":49152}]' | grep variant
  TCSPMV_LIB=$PWD/paper_1103_2405_b200/lib/$L timeout 600 python bench/explore_pb.py c3_flickr '[{"two_phase":0}]' | grep variant
done
done
for L in libtcspmv_prev.so libtcspmv.so; do TCSPMV_LIB=$PWD/paper_1103_2405_b200/lib/$L timeout 900 python bench/pr_c4.py; done
timeout 1800 python -m pytest tests/test_gpu_spmv.py tests/test_gpu_iter.py -q -x 2>&1 | tail -2
