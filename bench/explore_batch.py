"""Exploration: batched RWR (25 queries, f1) per-iteration time on a config; tiling of the batch
plan via TCSPMV_BATCH_TW / TCSPMV_BATCH_TILES."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import graphgen  # noqa: E402
from paper_1103_2405_b200 import Solver  # noqa: E402

G = graphgen.make_graph(sys.argv[1] if len(sys.argv) > 1 else "c2")
deg = np.diff(G.row_ptr) + np.bincount(G.col, minlength=G.n)
qs = np.random.default_rng(graphgen.SEED_QUERY).choice(np.nonzero(deg > 0)[0], size=25, replace=False)
for tw, tiles in json.loads(os.environ.get("BATCH_VARIANTS", "[[413696, 1]]")):
    os.environ["TCSPMV_BATCH_TW"] = str(tw)
    os.environ["TCSPMV_BATCH_TILES"] = str(tiles)
    s = Solver("rwr", G.n, G.row_ptr, G.col, device=0)
    t0 = time.time()
    s.run_batch(qs)
    b = time.time() - t0
    info = s.run_batch(qs)
    print(json.dumps(dict(tw=tw, tiles=tiles, it=info["iterations"], us_per_iter=round(info["us_per_iter"], 1),
                          first_call_s=round(b, 1))), flush=True)
    s.close()
