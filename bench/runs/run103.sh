# row-major units per lane per batch in the unstaged one-pass kernel: 1 (shipped) vs 2, after round 2's epilogue changes
for L in libtcspmv.so libtcspmv_ub2.so; do
  echo "lib $L"
  TCSPMV_LIB=$PWD/paper_1103_2405_b200/lib/$L VARIANTS='[{}]' timeout 600 python bench/explore_solver_plan.py c2 2>&1 | grep -v batch_fuse
  TCSPMV_LIB=$PWD/paper_1103_2405_b200/lib/$L timeout 600 python bench/explore_pb.py c2 '[{"two_phase":0}]' | grep variant
  TCSPMV_LIB=$PWD/paper_1103_2405_b200/lib/$L timeout 600 python bench/explore_pb.py c3_flickr '[{"two_phase":0}]' | grep variant
done
