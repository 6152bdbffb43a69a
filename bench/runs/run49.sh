O=gpurun_out/r49.jsonl; : > $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -Xcompiler -fPIC -shared -DPB_ET=1024 -DPB_RT=1024 bench/probe/pb_probe.cu -o bench/probe/libpb_probe.so
PB_C=16384 PB_RB=24576 timeout 300 python bench/probe/pb_probe.py c2 4 >> $O 2>>gpurun_out/r49.err
PB_C=16384 PB_RB=24576 timeout 300 python bench/probe/pb_probe.py c2 4 --pattern >> $O 2>>gpurun_out/r49.err
#PB_C=16384 PB_RB=24576 timeout 900 ncu --set full --import-source on --clock-control none --kernel-name regex:pb_ --launch-skip 8 -c 2 -o gpurun_out/r49_pb python bench/probe/pb_probe.py c2 4 > gpurun_out/r49.log 2>&1
