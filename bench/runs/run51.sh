# session-3 bench line + launch list + full capture of the dominant kernel (SASS stalls kept)
python bench.py > gpurun_out/r51_bench.json 2> gpurun_out/r51_bench.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r51_bench_reference.json 2>> gpurun_out/r51_bench.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --print-units base \
    --log-file gpurun_out/r51_launches_bench.csv python bench.py --steps 3 --warmup 3 --no-extras > gpurun_out/r51_ncu_list.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tc_spmv_tile -s 5 -c 1 -o gpurun_out/r51_full_bench \
    python bench.py --steps 3 --warmup 3 --no-extras > gpurun_out/r51_ncu_full.log 2>&1
