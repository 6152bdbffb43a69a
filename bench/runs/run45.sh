# probe v3: unrolled expand (2 CTAs/SM), float4 region loads, aligned regions
O=gpurun_out/r45.jsonl; : > $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -Xcompiler -fPIC -shared bench/probe/pb_probe.cu -o bench/probe/libpb_probe.so
for cfg in "16384 24576 4" "24576 24576 4" "16384 16384 4" "16384 24576 8"; do
  set -- $cfg
  PB_C=$1 PB_RB=$2 timeout 300 python bench/probe/pb_probe.py c2 $3 >> $O 2>>gpurun_out/r45.err
done
PB_C=16384 PB_RB=24576 timeout 300 python bench/probe/pb_probe.py c2 4 --pattern >> $O 2>>gpurun_out/r45.err
