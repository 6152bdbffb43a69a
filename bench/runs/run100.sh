# source-level stalls of the one-pass SpMV tile kernel (c2 valued, two_phase=0)
R=${R:-r02h}
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:tc_spmv_tile -s 3 -c 1 -o gpurun_out/${R}_s \
    python bench/explore_pb.py c2 '[{"two_phase":0}]' > gpurun_out/${R}_ncu.log 2>&1; echo ncu=$?
ncu -i gpurun_out/${R}_s.ncu-rep --page source --csv --print-units base > gpurun_out/${R}_src.csv 2>&1
rm -f gpurun_out/${R}_s.ncu-rep
