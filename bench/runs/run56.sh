# x relabel: scatter (default) vs gather form, c2 valued and pattern; then the GPU tests and smoke
O=gpurun_out/r56.jsonl; : > $O
python bench/explore_env.py c2 > /dev/null 2>&1
ENVS='[{}, {"TCSPMV_PERMUTE": "gather"}]' timeout 300 python bench/explore_env.py c2 >> $O 2>>gpurun_out/r56.err
ENVS='[{}, {"TCSPMV_PERMUTE": "gather"}]' timeout 300 python bench/explore_env.py c2 --pattern >> $O 2>>gpurun_out/r56.err
python -m pytest tests -m gpu -x -q > gpurun_out/r56_pytest.log 2>&1; echo pytest rc=$? >> gpurun_out/r56_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r56_smoke.log 2>&1; echo smoke rc=$? >> gpurun_out/r56_smoke.log
