# prefetch_rm: ent consulted only where it decides a load (current) vs the previous commit (prev)
for r in 1 2; do
for L in libtcspmv_prev.so libtcspmv.so; do
  echo "lib $L"
  TCSPMV_LIB=$PWD/paper_1103_2405_b200/lib/$L VARIANTS='[{}]' timeout 600 python bench/explore_solver_plan.py c2 2>&1 | grep -v batch_fuse
done
done
timeout 1200 python -m pytest tests/test_gpu_iter.py tests/test_gpu_loopback.py -q -x 2>&1 | tail -2
