nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -Xcompiler -fPIC -shared -DPB_RT=1024 -DPB_ET=1024 bench/probe/pb_probe.cu -o bench/probe/libpb_probe.so
PB_C=16384 PB_RB=24576 timeout 900 ncu --set full --import-source on --clock-control none --kernel-name regex:pb_ --launch-skip 8 -c 2 -o gpurun_out/r47_pb python bench/probe/pb_probe.py c2 4 > gpurun_out/r47.log 2>&1
ncu -i gpurun_out/r47_pb.ncu-rep --page raw --csv > gpurun_out/r47_raw.csv 2>&1
