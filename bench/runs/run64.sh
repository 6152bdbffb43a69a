# probe v8 sweep: row groups, chunk size, CTA sizes (overlapped phases)
O=gpurun_out/r64.jsonl; : > $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -Xcompiler -fPIC -shared -Ipaper_1103_2405_b200/csrc -DPB_ET=1024 -DPB_RT=1024 -DPB_CMAX=32768 bench/probe/pb_probe.cu -o bench/probe/libpb_probe.so
for cfg in "16384 24576 8" "16384 24576 6" "32768 24576 4" "32768 24576 8" "16384 32768 4"; do
  set -- $cfg
  PB_OVERLAP=1 PB_C=$1 PB_RB=$2 timeout 300 python bench/probe/pb_probe.py c2 $3 | sed "s/^{/{\"C\": $1, \"RB\": $2, /" >> $O 2>>gpurun_out/r64.err
done
