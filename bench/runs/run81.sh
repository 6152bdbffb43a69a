# compute-sanitizer over bench/sanitize_run.py (round-2 paths included: PDL chain, slices, batch)
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1500 $CS --tool memcheck --leak-check no python bench/sanitize_run.py c1 > gpurun_out/r02b_sanitize_memcheck.log 2>&1; echo memcheck=$?
timeout 1500 $CS --tool synccheck python bench/sanitize_run.py c1 > gpurun_out/r02b_sanitize_synccheck.log 2>&1; echo synccheck=$?
timeout 2400 $CS --tool racecheck --racecheck-report hazard python bench/sanitize_run.py t_small > gpurun_out/r02b_sanitize_racecheck.log 2>&1; echo racecheck=$?
timeout 1500 $CS --tool initcheck python bench/sanitize_run.py t_small > gpurun_out/r02b_sanitize_initcheck.log 2>&1; echo initcheck=$?
for f in gpurun_out/r02b_sanitize_*.log; do echo $f; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|hazard" $f | tail -2; done
