# feasibility probe: gather-free two-phase SpMV (bench/probe/pb_probe.*) on c2
O=gpurun_out/r43.jsonl; : > $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -Xcompiler -fPIC -shared bench/probe/pb_probe.cu -o bench/probe/libpb_probe.so
for cfg in "32768 49152 4" "16384 24576 4" "49152 49152 4" "32768 49152 2" "32768 49152 8"; do
  set -- $cfg
  PB_C=$1 PB_RB=$2 timeout 400 python bench/probe/pb_probe.py c2 $3 >> $O 2>>gpurun_out/r43.err
done
PB_C=32768 PB_RB=49152 timeout 400 python bench/probe/pb_probe.py c2 4 --pattern >> $O 2>>gpurun_out/r43.err
