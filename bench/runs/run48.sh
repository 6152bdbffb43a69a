# probe v5: flat flush (one step per 32 stage positions)
O=gpurun_out/r48.jsonl; : > $O
for v in "1024 1024" "512 512" "1024 512"; do
  set -- $v
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -Xcompiler -fPIC -shared -DPB_ET=$1 -DPB_RT=$2 bench/probe/pb_probe.cu -o bench/probe/libpb_probe.so
  PB_C=16384 PB_RB=24576 timeout 300 python bench/probe/pb_probe.py c2 4 | sed "s/^{/{\"et\": $1, \"rt\": $2, /" >> $O 2>>gpurun_out/r48.err
done
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -Xcompiler -fPIC -shared -DPB_ET=1024 -DPB_RT=1024 bench/probe/pb_probe.cu -o bench/probe/libpb_probe.so
PB_C=32768 PB_RB=24576 timeout 300 python bench/probe/pb_probe.py c2 4 >> $O 2>>gpurun_out/r48.err
PB_C=16384 PB_RB=24576 timeout 300 python bench/probe/pb_probe.py c2 8 >> $O 2>>gpurun_out/r48.err
PB_C=16384 PB_RB=24576 timeout 300 python bench/probe/pb_probe.py c2 4 --pattern >> $O 2>>gpurun_out/r48.err
