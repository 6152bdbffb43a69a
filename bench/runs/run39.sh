# BASELINE configs[3] (it-2004-shaped, 1.15B edges) on one B200: PageRank, full-size parity, SpMV tiling, HITS
C4_HITS=1 timeout 2400 python bench/experiment_c4.py > gpurun_out/r39_c4.jsonl 2> gpurun_out/r39_c4.err
free -g >> gpurun_out/r39_c4.err
