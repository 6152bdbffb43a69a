# source-level stalls of the batched RWR SpMM (c2, 25 queries, host-driven loop)
R=r02g
HOST_LOOP=1 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:spmm_rwr_tile -s 1 -c 1 -o gpurun_out/${R}_b \
    python bench/batch_once.py c2 2 > gpurun_out/${R}_ncu.log 2>&1; echo ncu=$?
ncu -i gpurun_out/${R}_b.ncu-rep --page source --csv --print-units base > gpurun_out/${R}_src.csv 2>&1
rm -f gpurun_out/${R}_b.ncu-rep
