# probe v4: batched run descriptors in the flush
O=gpurun_out/r46.jsonl; : > $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -Xcompiler -fPIC -shared bench/probe/pb_probe.cu -o bench/probe/libpb_probe.so
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -Xcompiler -fPIC -shared -DPB_RT=1024 -DPB_ET=1024 bench/probe/pb_probe.cu -o bench/probe/libpb_probe_1k.so
for cfg in "16384 24576 4" "24576 24576 4" "16384 24576 8"; do
  set -- $cfg
  PB_C=$1 PB_RB=$2 timeout 300 python bench/probe/pb_probe.py c2 $3 >> $O 2>>gpurun_out/r46.err
done
PB_C=16384 PB_RB=24576 timeout 300 python bench/probe/pb_probe.py c2 4 --pattern >> $O 2>>gpurun_out/r46.err
cp bench/probe/libpb_probe_1k.so bench/probe/libpb_probe.so
PB_C=16384 PB_RB=24576 timeout 300 python bench/probe/pb_probe.py c2 4 >> $O 2>>gpurun_out/r46.err
PB_C=32768 PB_RB=49152 timeout 300 python bench/probe/pb_probe.py c2 4 >> $O 2>>gpurun_out/r46.err
