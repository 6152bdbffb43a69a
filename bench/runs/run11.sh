export VARIANTS='[{"tile_width":24576,"num_tiles":1,"workload_size":1024}]'
ncu --set full --clock-control none --import-source on -k regex:tc_spmv_tile -s 6 -c 2 -o gpurun_out/prof_c2_v4 python bench/explore_spmv.py c2 > gpurun_out/ncu4.log 2>&1
ncu -i gpurun_out/prof_c2_v4.ncu-rep --page raw --csv > gpurun_out/prof_c2_v4_raw.csv 2>&1
ncu -i gpurun_out/prof_c2_v4.ncu-rep --page source --csv > gpurun_out/prof_c2_v4_src.csv 2>&1
ncu -i gpurun_out/prof_c2_v4.ncu-rep --page details --csv > gpurun_out/prof_c2_v4_details.csv 2>&1
python bench/calibrate.py --quick 2>&1 | tail -3
