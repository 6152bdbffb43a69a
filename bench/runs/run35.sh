# Round-1 re-entry check: GPU parity suite, the default bench line, the ncu launch list + full capture.
set -x
python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r35_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r35_smoke.log 2>&1; echo smoke=$? >> gpurun_out/r35_smoke.log
python bench.py > gpurun_out/r35_bench.json 2> gpurun_out/r35_bench.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r35_bench_ref.json 2> gpurun_out/r35_bench_ref.err
bash bench/ncu_bench.sh r35
