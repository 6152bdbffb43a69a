# source-level stall attribution of pb_spmv (ncu --page source), c2 valued bench command
R=r02c
TCSPMV_BENCH_NO_NCU=1 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:pb_spmv -s 5 -c 1 -o gpurun_out/${R}_full_bench \
    python bench.py --steps 3 --warmup 3 --no-extras > gpurun_out/${R}_ncu_full.log 2>&1; echo ncu=$?
ncu -i gpurun_out/${R}_full_bench.ncu-rep --page source --csv --print-units base --kernel-name regex:pb_spmv > gpurun_out/${R}_src.csv 2>&1
rm -f gpurun_out/${R}_full_bench.ncu-rep
wc -l gpurun_out/${R}_src.csv; head -3 gpurun_out/${R}_src.csv | cut -c1-600
