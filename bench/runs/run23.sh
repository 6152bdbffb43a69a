python -m pytest tests/test_gpu_iter.py -x -q -k "batch" 2>&1 | grep -vE "^\s+File|^    " | tail -3
python - <<'PY'
import json, numpy as np, sys
sys.path.insert(0, '.')
import graphgen
from paper_1103_2405_b200 import Solver
G = graphgen.make_graph("c2")
s = Solver("rwr", G.n, G.row_ptr, G.col, device=0, num_tiles=0, workload_size=1024)
deg = np.diff(G.row_ptr) + np.bincount(G.col, minlength=G.n)
rng = np.random.default_rng(graphgen.SEED_QUERY)
qs = rng.choice(np.nonzero(deg > 0)[0], size=25, replace=False)
s.run_batch(qs); info = s.run_batch(qs)
print(json.dumps(dict(batch=25, it=info["iterations"], us_per_iter=round(info["us_per_iter"],1), us_per_query_iter=round(info["us_per_iter"]/25,1))))
PY
