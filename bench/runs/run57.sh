python bench.py --steps 200 --warmup 5 --no-extras > gpurun_out/r57_bench.json 2> gpurun_out/r57.err
python -m pytest tests/test_gpu_spmv.py -m gpu -x -q -k "auto_and_deterministic" >> gpurun_out/r57.err 2>&1; echo pytest rc=$? >> gpurun_out/r57.err
