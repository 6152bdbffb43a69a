# Round-end profile of the bench command (one GPU): the launch list (per-launch duration and DRAM
# bytes, clocks not locked) and one full capture of the dominant kernel.  Output in gpurun_out/.
R=${1:-r01}
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --print-units base \
    --log-file gpurun_out/${R}_launches_bench.csv python bench.py --steps 3 --warmup 3 --no-extras > gpurun_out/${R}_ncu_list.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tc_spmv_tile -s 5 -c 1 -o gpurun_out/${R}_full_bench \
    python bench.py --steps 3 --warmup 3 --no-extras > gpurun_out/${R}_ncu_full.log 2>&1
ncu -i gpurun_out/${R}_full_bench.ncu-rep --page raw --csv --print-units base > gpurun_out/${R}_full_bench_raw.csv 2>&1
ncu -i gpurun_out/${R}_full_bench.ncu-rep --page source --csv --kernel-name regex:tc_spmv_tile --launch-skip 0 --launch-count 1 \
    > gpurun_out/${R}_full_bench_src.csv 2>&1
rm -f gpurun_out/${R}_full_bench.ncu-rep
