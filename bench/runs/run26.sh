timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
export VARIANTS='[{"num_tiles":0,"workload_size":256},{"num_tiles":0,"workload_size":512},{"num_tiles":0,"workload_size":1024},{"tile_width":49152,"num_tiles":2,"workload_size":512}]'
for lib in libtcspmv.so libtcspmv_static.so; do
  echo "== $lib"
  TCSPMV_LIB=$PWD/paper_1103_2405_b200/lib/$lib python bench/explore_spmv.py c2 2>&1 | tail -4 | cut -c1-110
  TCSPMV_LIB=$PWD/paper_1103_2405_b200/lib/$lib python bench/explore_spmv.py c2 --pattern 2>&1 | tail -4 | cut -c1-110
done
python bench/experiment_autotune.py --quick > gpurun_out/r01_autotune_dyn.json 2> gpurun_out/r01_autotune_dyn.err; cut -c1-330 gpurun_out/r01_autotune_dyn.err | tail -6
