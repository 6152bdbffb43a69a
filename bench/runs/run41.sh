bash bench/runs/run40.sh
timeout 1800 python bench/experiment_c4_tiles.py > gpurun_out/r41_c4_tiles.jsonl 2> gpurun_out/r41_c4_tiles.err
