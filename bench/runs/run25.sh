python -m pytest tests/test_gpu_iter.py -x -q -k "config0" 2>&1 | grep -vE "^\s+File|^    " | tail -3
python bench/experiment_autotune.py --quick > gpurun_out/r01_autotune.json 2> gpurun_out/r01_autotune.err; tail -8 gpurun_out/r01_autotune.err | cut -c1-400
