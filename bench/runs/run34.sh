export VARIANTS='[{"num_tiles":0,"workload_size":1024}]'
L=$PWD/paper_1103_2405_b200/lib
for lib in libtcspmv.so libtcspmv_rmub2.so libtcspmv_cmv4.so libtcspmv_rmcm.so; do
  echo "== $lib"
  export TCSPMV_LIB=$L/$lib
  python bench/explore_spmv.py c2 2>&1 | tail -1 | cut -c1-90
  python bench/explore_spmv.py c2 --pattern 2>&1 | tail -1 | cut -c1-90
  python bench/experiment_f4.py 2>/dev/null | cut -c1-140
  python bench/explore_pr.py c2 2>&1 | head -1 | cut -c1-120
done
unset TCSPMV_LIB
export BATCH_VARIANTS='[[413696, 0], [413696, 1], [262144, 1], [131072, 2], [524288, 1]]'
python bench/explore_batch.py c2
