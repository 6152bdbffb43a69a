export VARIANTS='[{"num_tiles":0,"workload_size":1024}]'
L=$PWD/paper_1103_2405_b200/lib
ncu_dram() { ncu --metrics dram__bytes_read.sum,lts__t_sector_hit_rate.pct -k regex:tc_spmv_tile -s 3 -c 1 --csv --print-units base \
      --cache-control none python bench/explore_spmv.py c2 2>/dev/null | grep -E "dram__bytes_read|lts__t_sector_hit" | awk -F'","' '{print $(NF-2), $NF}'; }
for cfg in "libtcspmv.so 0" "libtcspmv_pf1x.so 0" "libtcspmv_pf1x.so 20" "libtcspmv_pf1x.so 40" "libtcspmv_pf0x.so 0" "libtcspmv_pf0x.so 20"; do
  set -- $cfg
  echo "== $1 window=$2"
  export TCSPMV_LIB=$L/$1
  if [ "$2" != "0" ]; then export TCSPMV_L2_WINDOW=$2; else unset TCSPMV_L2_WINDOW; fi
  python bench/explore_spmv.py c2 2>&1 | tail -1 | cut -c1-90
  python bench/explore_spmv.py c2 --pattern 2>&1 | tail -1 | cut -c1-90
  ncu_dram
  python bench/explore_pr.py c2 2>&1 | cut -c1-120
done
