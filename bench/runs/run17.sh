python -m pytest tests -m gpu -x -q 2>&1 | grep -vE "^\s+File|^    " | tail -5
python bench.py --steps 200 --warmup 10 > gpurun_out/bench_r01.json 2> gpurun_out/bench_r01.err; tail -2 gpurun_out/bench_r01.err; cat gpurun_out/bench_r01.json
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 30 -c 12 --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 4 --warmup 3 --no-extras > /dev/null 2>&1
export VARIANTS='[{}]'
ncu --set full --clock-control none --import-source on -k regex:tc_spmv_tile -s 8 -c 2 -o gpurun_out/prof_r01 python bench/explore_spmv.py c2 > /dev/null 2>&1
ncu -i gpurun_out/prof_r01.ncu-rep --page raw --csv > gpurun_out/prof_r01_raw.csv 2>&1
ncu -i gpurun_out/prof_r01.ncu-rep --page details --csv > gpurun_out/prof_r01_details.csv 2>&1
