# probe v10: persistent reduce with TMA bulk double-buffered regions
O=gpurun_out/r63.jsonl; : > $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -Xcompiler -fPIC -shared -Ipaper_1103_2405_b200/csrc -DPB_ET=1024 -DPB_RT=1024 bench/probe/pb_probe.cu -o bench/probe/libpb_probe.so
for rb in 24576 16384; do
  PB_PIPE=1 PB_OVERLAP=1 PB_C=16384 PB_RB=$rb timeout 300 python bench/probe/pb_probe.py c2 4 | sed "s/^{/{\"rb\": $rb, \"pipe\": 1, /" >> $O 2>>gpurun_out/r63.err
done
PB_PIPE=1 PB_OVERLAP=1 PB_C=16384 PB_RB=24576 timeout 300 python bench/probe/pb_probe.py c2 4 --pattern | sed "s/^{/{\"pipe\": 1, /" >> $O 2>>gpurun_out/r63.err
