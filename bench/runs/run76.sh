# batched RWR: fused Eq. 9 (per-workload post-pass) vs the separate pass; parity tests of the batch path
timeout 300 python -m pytest tests/test_gpu_iter.py -q -x -k "batch" 2>&1 | tail -3
VARIANTS='[]' timeout 300 python bench/explore_solver_plan.py c2 2>&1
