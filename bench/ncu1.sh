set -x
export VARIANTS='[{"num_tiles":0,"workload_size":1024},{"tile_width":49152,"num_tiles":1,"workload_size":1024}]'
ncu --set full --clock-control none --import-source on -k regex:tc_spmv_tile -s 6 -c 4 -o gpurun_out/prof_c2_v1 python bench/explore_spmv.py c2 > gpurun_out/ncu1.log 2>&1
ncu -i gpurun_out/prof_c2_v1.ncu-rep --page raw --csv > gpurun_out/prof_c2_v1_raw.csv 2>&1
python -m pytest tests -m gpu -x -q 2>&1 | tail -15
