python bench/calibrate.py --quick 2>&1 | tail -1
cp gpurun_out/perf_table_b200.json paper_1103_2405_b200/data/perf_table_b200.json
export VARIANTS='[{"num_tiles":0,"workload_size":1024},{}]'
for hot in 2147483647 16384 49152 131072; do echo "== hot $hot"; TCSPMV_L1_HOT=$hot python bench/explore_spmv.py c2 2>&1 | tail -2 | cut -c1-200; done
python bench/explore_pr.py c2 2>&1 | tail -6
