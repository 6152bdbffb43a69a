# row entry / epilogue operands taken over after the unit's gathers (current) vs at the row start (prev)
for r in 1 2; do
for L in libtcspmv_prev.so libtcspmv.so; do
  echo "lib $L"
  TCSPMV_LIB=$PWD/paper_1103_2405_b200/lib/$L VARIANTS='[{}]' timeout 600 python bench/explore_solver_plan.py c2 2>&1 | grep -v batch_fuse
  TCSPMV_LIB=$PWD/paper_1103_2405_b200/lib/$L timeout 600 python bench/explore_pb.py c2 '[{"two_phase":0}]' | grep variant
  TCSPMV_LIB=$PWD/paper_1103_2405_b200/lib/$L timeout 600 python bench/explore_pb.py c3_flickr '[{"two_phase":0}]' | grep variant
done
done
timeout 1500 python -m pytest tests/test_gpu_spmv.py tests/test_gpu_iter.py -q -x 2>&1 | tail -1
