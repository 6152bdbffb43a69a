# ncu --set full metrics of the one-pass tile kernel after round 2 (c2 valued, two_phase=0)
R=r02j
timeout 1200 ncu --set full --clock-control none -k regex:tc_spmv_tile -s 3 -c 1 -o gpurun_out/${R}_s \
    python bench/explore_pb.py c2 '[{"two_phase":0}]' > gpurun_out/${R}_ncu.log 2>&1; echo ncu=$?
ncu -i gpurun_out/${R}_s.ncu-rep --page raw --csv --print-units base > gpurun_out/${R}_raw.csv 2>&1
rm -f gpurun_out/${R}_s.ncu-rep
