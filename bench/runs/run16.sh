export VARIANTS='[{"num_tiles":0,"workload_size":1024},{"tile_width":49152,"num_tiles":1,"workload_size":1024},{"tile_width":49152,"num_tiles":2,"workload_size":1024},{"tile_width":49152,"num_tiles":4,"workload_size":1024},{"tile_width":24576,"num_tiles":3,"workload_size":1024}]'
python bench/explore_spmv.py c2 2>&1 | tail -5 | cut -c1-150
python bench/explore_spmv.py c2 --pattern 2>&1 | tail -5 | cut -c1-150
python bench/calibrate.py --quick 2>&1 | tail -2
