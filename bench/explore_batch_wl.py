"""Batched RWR (25 queries, c2): the batch plan's workload size (it follows the solver's WL)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import graphgen  # noqa: E402
from paper_1103_2405_b200 import Solver  # noqa: E402

G = graphgen.make_graph("c2")
deg = np.diff(G.row_ptr) + np.bincount(G.col, minlength=G.n)
qs = np.random.default_rng(graphgen.SEED_QUERY).choice(np.nonzero(deg > 0)[0], size=25, replace=False)
for wl in [128, 256, 512, 1024, 2048, 4096]:
    s = Solver("rwr", G.n, G.row_ptr, G.col, device=0, workload_size=wl)
    s.run_batch(qs)
    b = s.run_batch(qs)
    print(json.dumps(dict(wl=wl, it=b["iterations"], us_per_iter=round(b["us_per_iter"], 1),
                          query_iters_per_s=round(25e6 / b["us_per_iter"], 1))), flush=True)
    s.close()
