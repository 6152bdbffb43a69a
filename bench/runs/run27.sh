export VARIANTS='[{"num_tiles":0,"workload_size":256},{"num_tiles":0,"workload_size":512},{"num_tiles":0,"workload_size":1024}]'
summ() { python -c "
import json,sys
for r in json.load(sys.stdin): print(r['graph'], r['alpha'], [(g['wl'], g['us'], g['predicted_us']) for g in r['grid']])"; }
for lib in libtcspmv.so libtcspmv_dyn1.so libtcspmv_dyn3.so libtcspmv_static.so; do
  echo "== $lib"
  export TCSPMV_LIB=$PWD/paper_1103_2405_b200/lib/$lib
  python bench/explore_spmv.py c2 2>&1 | tail -3 | cut -c1-80
  python bench/explore_spmv.py c2 --pattern 2>&1 | tail -3 | cut -c1-80
  python bench/experiment_autotune.py --quick --t0 --graph youtube 2>/dev/null | summ
  python bench/experiment_autotune.py --quick --t0 --graph flickr 2>/dev/null | summ
done
