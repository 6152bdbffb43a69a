# batched RWR: branch-free x-row loads (zero row for the sentinel) vs the select (prev)
for r in 1 2; do
for L in libtcspmv_prev.so libtcspmv.so; do
  echo "lib $L"
  TCSPMV_LIB=$PWD/paper_1103_2405_b200/lib/$L timeout 600 python bench/explore_batch_wl.py 2>&1 | grep '"wl": 1024'
done
done
timeout 900 python -m pytest tests/test_gpu_iter.py -q -x -k batch 2>&1 | tail -2
