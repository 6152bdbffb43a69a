# ncu of the c4 auto plan's tile launches (first SpMV skipped): DRAM-served x gathers
timeout 2400 ncu --set full --clock-control none -k regex:tc_spmv_tile -s 5 -c 5 -o gpurun_out/r74_c4 python bench/ncu_c4.py > gpurun_out/r74.log 2>&1
ncu -i gpurun_out/r74_c4.ncu-rep --page raw --csv --print-units base > gpurun_out/r74_raw.csv 2>&1
rm -f gpurun_out/r74_c4.ncu-rep
