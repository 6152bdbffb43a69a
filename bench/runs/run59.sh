# probe v7: expand of group g+1 overlapping the reduce of group g (two streams, two buffers)
O=gpurun_out/r59.jsonl; : > $O
for v in "1024 1024" "512 512"; do
  set -- $v
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -Xcompiler -fPIC -shared -DPB_ET=$1 -DPB_RT=$2 bench/probe/pb_probe.cu -o bench/probe/libpb_probe.so
  for G in 4 8; do
    PB_OVERLAP=1 PB_C=16384 PB_RB=24576 timeout 300 python bench/probe/pb_probe.py c2 $G | sed "s/^{/{\"et\": $1, /" >> $O 2>>gpurun_out/r59.err
  done
done
PB_OVERLAP=0 PB_C=16384 PB_RB=24576 timeout 300 python bench/probe/pb_probe.py c2 4 >> $O 2>>gpurun_out/r59.err
