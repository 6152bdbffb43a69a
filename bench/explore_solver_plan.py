"""Exploration: the solvers' plan choice on c2 (tuner candidates R21, orientation) against fixed
settings, and batched RWR with / without the fused Eq. 9 (TCSPMV_BATCH_FUSE)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import graphgen  # noqa: E402
from paper_1103_2405_b200 import Solver  # noqa: E402

G = graphgen.make_graph(sys.argv[1] if len(sys.argv) > 1 else "c2")
variants = json.loads(os.environ.get("VARIANTS", '[{}, {"orient": 0}, {"orient": 0, "workload_size": 1024}, {"workload_size": 1024}]'))
for algo in ("pagerank", "hits", "rwr"):
    for kw in variants:
        s = Solver(algo, G.n, G.row_ptr, G.col, device=0, **kw)
        st = s.stats()
        s.run(5 if algo == "rwr" else 0)
        info = s.run(5 if algo == "rwr" else 0)
        print(json.dumps(dict(algo=algo, opts=kw, us_per_iter=round(info["us_per_iter"], 1),
                              predicted=round(info["predicted_us_per_iter"], 1), it=info["iterations"],
                              orient=st["orient"], wl=st["wl"], tiles=st["num_tiles"], tw=st["tile_width"],
                              two_phase=st["two_phase"])), flush=True)
        s.close()
deg = np.diff(G.row_ptr) + np.bincount(G.col, minlength=G.n)
qs = np.random.default_rng(graphgen.SEED_QUERY).choice(np.nonzero(deg > 0)[0], size=25, replace=False)
for fuse in ("1", "0"):
    os.environ["TCSPMV_BATCH_FUSE"] = fuse
    s = Solver("rwr", G.n, G.row_ptr, G.col, device=0)
    s.run_batch(qs)
    b = s.run_batch(qs)
    print(json.dumps(dict(batch_fuse=fuse, it=b["iterations"], us_per_iter=round(b["us_per_iter"], 1),
                          query_iters_per_s=round(25e6 / b["us_per_iter"], 1))), flush=True)
    s.close()
