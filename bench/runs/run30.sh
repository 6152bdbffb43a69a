timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
export VARIANTS='[{"num_tiles":0,"workload_size":512},{"num_tiles":0,"workload_size":1024}]'
summ() { python -c "
import json,sys
for r in json.load(sys.stdin): print(r['graph'], r['alpha'], [(g['wl'], g['us'], g['predicted_us']) for g in r['grid']])"; }
python bench/explore_spmv.py c2 2>&1 | tail -2 | cut -c1-80
python bench/explore_spmv.py c2 --pattern 2>&1 | tail -2 | cut -c1-80
python bench/experiment_autotune.py --quick > gpurun_out/r01_autotune.json 2> gpurun_out/r01_autotune.err; cut -c1-330 gpurun_out/r01_autotune.err | tail -6
python bench.py > gpurun_out/r01_bench.json 2> gpurun_out/r01_bench.err; tail -c 3000 gpurun_out/r01_bench.json
bash bench/ncu_bench.sh r01
ls gpurun_out
