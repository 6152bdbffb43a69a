./bench/probe/probe3 > gpurun_out/r01_probe_tma_gather4.jsonl 2>&1; cat gpurun_out/r01_probe_tma_gather4.jsonl
bash bench/runs/run27.sh
