timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
export VARIANTS='[{"num_tiles":0,"workload_size":1024},{"num_tiles":0,"workload_size":512}]'
L=$PWD/paper_1103_2405_b200/lib
summ() { python -c "
import json,sys
for r in json.load(sys.stdin): print(r['graph'], r['alpha'], [(g['wl'], g['us'], g['predicted_us']) for g in r['grid']])"; }
for lib in libtcspmv.so libtcspmv_pfn.so libtcspmv_pf0nox.so libtcspmv_dyn0.so; do
  echo "== $lib"
  export TCSPMV_LIB=$L/$lib
  python bench/explore_spmv.py c2 2>&1 | tail -2 | cut -c1-90
  python bench/explore_spmv.py c2 --pattern 2>&1 | tail -2 | cut -c1-90
  python bench/experiment_autotune.py --quick --t0 --graph youtube 2>/dev/null | summ
done
unset TCSPMV_LIB
python bench/experiment_f4.py > gpurun_out/r01_f4_dense_banded.json 2> gpurun_out/f4.err; cat gpurun_out/r01_f4_dense_banded.json | cut -c1-250
python bench/experiment_f2.py c2 c3_flickr > gpurun_out/r01_f2_ablation.json 2> gpurun_out/f2.err; cut -c1-250 gpurun_out/f2.err | tail -20
