# probe v2: heavy rows (CTA / warp per row) + phase split
O=gpurun_out/r44.jsonl; : > $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -Xcompiler -fPIC -shared bench/probe/pb_probe.cu -o bench/probe/libpb_probe.so
PB_C=16384 PB_RB=24576 timeout 300 python bench/probe/pb_probe.py c2 4 >> $O 2>>gpurun_out/r44.err
PB_C=32768 PB_RB=49152 timeout 300 python bench/probe/pb_probe.py c2 4 >> $O 2>>gpurun_out/r44.err
PB_C=32768 PB_RB=49152 timeout 300 python bench/probe/pb_probe.py c2 4 --pattern >> $O 2>>gpurun_out/r44.err
