"""Exploration: PageRank / HITS / RWR per-iteration time on c2 for given options."""
import json, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import graphgen
from paper_1103_2405_b200 import Solver
G = graphgen.make_graph(sys.argv[1] if len(sys.argv) > 1 else "c2")
variants = json.loads(os.environ.get("VARIANTS", "null")) or [dict(num_tiles=0, workload_size=1024)]
for algo in ("pagerank", "rwr", "hits"):
    for v in variants:
        t0 = time.time()
        s = Solver(algo, G.n, G.row_ptr, G.col, device=0, **v)
        b = time.time() - t0
        q = int(np.nonzero(np.diff(G.row_ptr) > 0)[0][0])
        s.run(q)
        info = s.run(q)
        st = s.stats()
        print(json.dumps(dict(algo=algo, opt=v, it=info["iterations"], us_per_iter=round(info["us_per_iter"], 1),
                              build_s=round(b, 1), launches=s.launches_per_iter, tiles=st["num_tiles"], wl=st["wl"])), flush=True)
        s.close()
