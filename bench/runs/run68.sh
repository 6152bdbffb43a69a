# probe v12: persistent TMA-pipelined reduce with two CTAs per SM (smaller bins)
O=gpurun_out/r68.jsonl; : > $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -Xcompiler -fPIC -shared -Ipaper_1103_2405_b200/csrc -DPB_ET=1024 -DPB_RT=1024 -DPB_PIPE_CTAS=2 bench/probe/pb_probe.cu -o bench/probe/libpb_probe.so
for rb in 12288 8192; do
  PB_PIPE=1 PB_OVERLAP=1 PB_C=16384 PB_RB=$rb timeout 300 python bench/probe/pb_probe.py c2 4 | sed "s/^{/{\"rb\": $rb, \"pipe_ctas\": 2, /" >> $O 2>>gpurun_out/r68.err
done
PB_PIPE=0 PB_OVERLAP=1 PB_C=16384 PB_RB=12288 timeout 300 python bench/probe/pb_probe.py c2 4 | sed "s/^{/{\"rb\": 12288, \"pipe\": 0, /" >> $O 2>>gpurun_out/r68.err
