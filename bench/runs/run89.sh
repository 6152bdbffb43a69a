# source-level stall attribution of the one-pass tile kernel inside the PageRank iteration (c2)
R=${R:-r02d}
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:tc_spmv_tile -s 2 -c 1 -o gpurun_out/${R}_pr \
    python bench/pr_once.py c2 > gpurun_out/${R}_ncu.log 2>&1; echo ncu=$?
ncu -i gpurun_out/${R}_pr.ncu-rep --page source --csv --print-units base > gpurun_out/${R}_src.csv 2>&1
ncu -i gpurun_out/${R}_pr.ncu-rep --page raw --csv --print-units base > gpurun_out/${R}_raw.csv 2>&1
rm -f gpurun_out/${R}_pr.ncu-rep
wc -l gpurun_out/${R}_src.csv
