export VARIANTS='[{"tile_width":49152,"num_tiles":1,"workload_size":1024}]'
ncu --set full --clock-control none --import-source on -k regex:tc_spmv_tile -s 6 -c 2 -o gpurun_out/prof_c2_v3 python bench/explore_spmv.py c2 > gpurun_out/ncu3.log 2>&1
ncu -i gpurun_out/prof_c2_v3.ncu-rep --page raw --csv > gpurun_out/prof_c2_v3_raw.csv 2>&1
ncu -i gpurun_out/prof_c2_v3.ncu-rep --page source --csv > gpurun_out/prof_c2_v3_src.csv 2>&1
ncu -i gpurun_out/prof_c2_v3.ncu-rep --page details --csv > gpurun_out/prof_c2_v3_details.csv 2>&1
export VARIANTS='[{"num_tiles":0,"workload_size":1024},{"tile_width":49152,"num_tiles":1,"workload_size":1024},{"tile_width":24576,"num_tiles":3,"workload_size":1024}]'
TCSPMV_LIB=$PWD/paper_1103_2405_b200/lib/libtcspmv_t768.so python bench/explore_spmv.py c2 2>&1 | tail -3
