export VARIANTS='[{"num_tiles":0,"workload_size":1024},{"num_tiles":0,"workload_size":512}]'
for lib in libtcspmv.so libtcspmv_xpol.so libtcspmv_pfpol.so libtcspmv_both.so libtcspmv_pf1.so libtcspmv_pf1x.so; do
  echo "== $lib"
  export TCSPMV_LIB=$PWD/paper_1103_2405_b200/lib/$lib
  python bench/explore_spmv.py c2 2>&1 | tail -2 | cut -c1-90
  python bench/explore_spmv.py c2 --pattern 2>&1 | tail -2 | cut -c1-90
  ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct -k regex:tc_spmv_tile -s 3 -c 1 --csv --print-units base \
      python bench/explore_spmv.py c2 2>/dev/null | grep -E "dram__bytes_read|lts__t_sector_hit|gpu__time" | awk -F'","' '{print $(NF-2), $NF}'
done
