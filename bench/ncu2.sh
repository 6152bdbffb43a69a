export VARIANTS='[{"tile_width":49152,"num_tiles":1,"workload_size":1024}]'
ncu --set full --clock-control none --import-source on -k regex:tc_spmv_tile -s 6 -c 4 -o gpurun_out/prof_c2_v2 python bench/explore_spmv.py c2 > gpurun_out/ncu2.log 2>&1
ncu -i gpurun_out/prof_c2_v2.ncu-rep --page raw --csv > gpurun_out/prof_c2_v2_raw.csv 2>&1
ncu -i gpurun_out/prof_c2_v2.ncu-rep --page source --csv --kernel-name regex:tc_spmv_tile --launch-skip 0 --launch-count 1 > gpurun_out/prof_c2_v2_src.csv 2>&1
python -m pytest tests/test_gpu_iter.py -x -q 2>&1 | tail -25
