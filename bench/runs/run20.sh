python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
python bench.py > gpurun_out/bench_r01.json 2> gpurun_out/bench_r01.err; tail -2 gpurun_out/bench_r01.err; cat gpurun_out/bench_r01.json
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_r01_ref.json 2>&1; cat gpurun_out/bench_r01_ref.json
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 30 -c 8 --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 4 --warmup 3 --no-extras > /dev/null 2>&1
export VARIANTS='[{}]'
ncu --set full --clock-control none --import-source on -k regex:tc_spmv_tile -s 4 -c 1 -o gpurun_out/prof_r01b python bench/explore_spmv.py c2 > /dev/null 2>&1
ncu -i gpurun_out/prof_r01b.ncu-rep --page raw --csv > gpurun_out/prof_r01b_raw.csv 2>&1
ncu -i gpurun_out/prof_r01b.ncu-rep --page source --csv > gpurun_out/prof_r01b_src.csv 2>&1
ncu -i gpurun_out/prof_r01b.ncu-rep --page details --csv > gpurun_out/prof_r01b_details.csv 2>&1
