python bench/calibrate.py --quick 2>&1 | tail -1
cp gpurun_out/perf_table_b200.json paper_1103_2405_b200/data/perf_table_b200.json
python -m pytest tests -m gpu -x -q 2>&1 | grep -vE "^\s+File|^    " | tail -4
export VARIANTS='[{"num_tiles":0,"workload_size":1024},{}]'
python bench/explore_spmv.py c2 2>&1 | tail -2 | cut -c1-200
python bench/explore_spmv.py c2 --pattern 2>&1 | tail -2 | cut -c1-200
python bench/explore_pr.py c2 2>&1 | tail -6
