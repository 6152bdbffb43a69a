"""Batched RWR (25 queries) on c2 for a few fixed iterations (ncu captures of spmm_rwr_tile)."""
import os, sys, json
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import graphgen
import paper_1103_2405_b200 as pkg
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2
G = graphgen.make_graph(cfg)
deg = np.diff(G.row_ptr) + np.bincount(G.col, minlength=G.n)
rng = np.random.default_rng(graphgen.SEED_QUERY)
qs = rng.choice(np.nonzero(deg > 0)[0], size=25, replace=False)
s = pkg.Solver("rwr", G.n, G.row_ptr, G.col, device=0, iter_kw=dict(fixed_iters=iters, host_loop=int(os.environ.get("HOST_LOOP", "1"))))
s.run_batch(qs)
info = s.run_batch(qs)
print(json.dumps(dict(us_per_iter=info["us_per_iter"], q_it_s=25e6 / info["us_per_iter"])))
