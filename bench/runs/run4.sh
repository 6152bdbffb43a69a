python -m pytest tests/test_gpu_iter.py tests/test_gpu_spmv.py -x -q 2>&1 | tail -15
export VARIANTS='[{"num_tiles":0,"workload_size":1024},{"num_tiles":0,"workload_size":4096},{"tile_width":49152,"num_tiles":1,"workload_size":1024},{"tile_width":49152,"num_tiles":1,"workload_size":1024,"stage_x":0},{"tile_width":49152,"num_tiles":3,"workload_size":1024},{"tile_width":49152,"num_tiles":8,"workload_size":1024}]'
python bench/explore_spmv.py c2 2>&1 | tail -8
python bench/explore_spmv.py c2 --pattern 2>&1 | tail -8
