# prefetch_rm with a real branch on has_acc (current) vs merged predicate (prev); c2 solvers twice, c4 PageRank
for r in 1 2; do
for L in libtcspmv_prev.so libtcspmv.so; do
  echo "lib $L"
  TCSPMV_LIB=$PWD/paper_1103_2405_b200/lib/$L VARIANTS='[{}]' timeout 600 python bench/explore_solver_plan.py c2 2>&1 | grep -v batch_fuse
done
done
for L in libtcspmv_prev.so libtcspmv.so; do TCSPMV_LIB=$PWD/paper_1103_2405_b200/lib/$L timeout 900 python bench/pr_c4.py; done
timeout 1200 python -m pytest tests/test_gpu_iter.py -q -x 2>&1 | tail -2
