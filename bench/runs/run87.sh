# full ncu capture of the dominant kernel (pb_spmv, x segment cap 6144) in the bench command
R=r02b
TCSPMV_BENCH_NO_NCU=1 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:pb_spmv -s 5 -c 1 -o gpurun_out/${R}_full_bench \
    python bench.py --steps 3 --warmup 3 --no-extras > gpurun_out/${R}_ncu_full.log 2>&1; echo ncu=$?
ncu -i gpurun_out/${R}_full_bench.ncu-rep --page raw --csv --print-units base > gpurun_out/${R}_full_bench_raw.csv 2>&1
ncu -i gpurun_out/${R}_full_bench.ncu-rep --page details --csv --print-units base > gpurun_out/${R}_full_bench_details.csv 2>&1
rm -f gpurun_out/${R}_full_bench.ncu-rep
wc -c gpurun_out/${R}_full_bench_raw.csv
