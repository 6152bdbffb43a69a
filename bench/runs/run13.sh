python -m pytest tests/test_gpu_spmv.py tests/test_gpu_iter.py tests/test_gpu_dist.py -x -q 2>&1 | tail -4
python bench.py --steps 200 --warmup 10 > gpurun_out/bench_r01_try.json 2> gpurun_out/bench_r01_try.err; tail -3 gpurun_out/bench_r01_try.err; cat gpurun_out/bench_r01_try.json
export VARIANTS='[{"num_tiles":0,"workload_size":1024}]'
TCSPMV_KERNEL=stream ncu --set full --clock-control none --import-source on -k regex:tc_spmv_wstream -s 3 -c 1 -o gpurun_out/prof_ws python bench/explore_spmv.py c2 > gpurun_out/ncu_ws.log 2>&1
ncu -i gpurun_out/prof_ws.ncu-rep --page raw --csv > gpurun_out/prof_ws_raw.csv 2>&1
ncu -i gpurun_out/prof_ws.ncu-rep --page source --csv > gpurun_out/prof_ws_src.csv 2>&1
