# prefetch_rm for entry-state epilogues only: timings vs base, then the GPU parity suite
for L in libtcspmv_base.so libtcspmv.so; do
  echo "lib $L"
  TCSPMV_LIB=$PWD/paper_1103_2405_b200/lib/$L VARIANTS='[{}]' timeout 600 python bench/explore_solver_plan.py c2 2>&1 | grep -v batch_fuse
  TCSPMV_LIB=$PWD/paper_1103_2405_b200/lib/$L timeout 600 python bench/explore_pb.py c2 '[{"two_phase":0}]' | grep variant
done
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
