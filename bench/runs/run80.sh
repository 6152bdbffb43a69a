# round-2 checkpoint: full GPU suite, smoke, bench line, reference arm, launch list of the bench command
timeout 2400 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/r02_gputest.log 2>&1; echo gputest=$? >> gpurun_out/r02_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1; echo smoke=$? >> gpurun_out/r02_smoke.log
timeout 1200 python bench.py > gpurun_out/r02_bench.log 2>&1; echo bench=$? >> gpurun_out/r02_bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02_bench_reference.log 2>&1
TCSPMV_BENCH_NO_NCU=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --print-units base \
    --log-file gpurun_out/r02_launches_bench.csv python bench.py --steps 3 --warmup 3 --no-extras > gpurun_out/r02_ncu_list.log 2>&1; echo ncu=$? >> gpurun_out/r02_ncu_list.log
tail -3 gpurun_out/r02_gputest.log; tail -2 gpurun_out/r02_smoke.log; tail -c 600 gpurun_out/r02_bench.log; tail -1 gpurun_out/r02_ncu_list.log
