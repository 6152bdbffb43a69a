# probe v11: static run index per stage position (no run search in the flush)
O=gpurun_out/r66.jsonl; : > $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -Xcompiler -fPIC -shared -Ipaper_1103_2405_b200/csrc -DPB_FLAT=2 -DPB_ET=1024 -DPB_RT=1024 bench/probe/pb_probe.cu -o bench/probe/libpb_probe.so
PB_OVERLAP=1 PB_C=16384 PB_RB=24576 timeout 300 python bench/probe/pb_probe.py c2 4 >> $O 2>>gpurun_out/r66.err
PB_OVERLAP=1 PB_C=16384 PB_RB=24576 timeout 300 python bench/probe/pb_probe.py c2 4 --pattern >> $O 2>>gpurun_out/r66.err
PB_OVERLAP=1 PB_C=16384 PB_RB=24576 timeout 300 python bench/probe/pb_probe.py c2 8 >> $O 2>>gpurun_out/r66.err
