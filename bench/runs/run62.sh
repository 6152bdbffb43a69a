# probe v9: reduce stages its position block in shared memory with the region
O=gpurun_out/r62.jsonl; : > $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -Xcompiler -fPIC -shared -DPB_ET=1024 -DPB_RT=1024 bench/probe/pb_probe.cu -o bench/probe/libpb_probe.so
for rb in 24576 16384; do
  PB_OVERLAP=1 PB_C=16384 PB_RB=$rb timeout 300 python bench/probe/pb_probe.py c2 4 | sed "s/^{/{\"rb\": $rb, /" >> $O 2>>gpurun_out/r62.err
done
PB_OVERLAP=1 PB_C=16384 PB_RB=16384 timeout 300 python bench/probe/pb_probe.py c2 4 --pattern >> $O 2>>gpurun_out/r62.err
