# one-pass tiles: entry-order epilogue state requested with the row entry (prefetch_rm) vs before (base)
for r in 1 2; do
for L in libtcspmv_base.so libtcspmv.so; do
  echo "lib $L"
  TCSPMV_LIB=$PWD/paper_1103_2405_b200/lib/$L VARIANTS='[{}]' timeout 600 python bench/explore_solver_plan.py c2 2>&1 | grep -v batch_fuse
  TCSPMV_LIB=$PWD/paper_1103_2405_b200/lib/$L timeout 600 python bench/explore_pb.py c2 '[{"two_phase":0}]' | grep variant
  TCSPMV_LIB=$PWD/paper_1103_2405_b200/lib/$L timeout 600 python bench/explore_pb.py c3_flickr '[{"two_phase":0}]' | grep variant
done
done
