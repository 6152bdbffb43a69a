"""Solver iteration time over plan variants: python bench/explore_solver.py c2 pagerank '[{...}, ...]'"""
import json, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import graphgen
import paper_1103_2405_b200 as pkg
cfg, algo = sys.argv[1], sys.argv[2]
variants = json.loads(sys.argv[3]) if len(sys.argv) > 3 else [dict(two_phase=0), dict(two_phase=1)]
G = graphgen.make_graph(cfg)
q = int(np.nonzero(np.diff(G.row_ptr) > 0)[0][0])
for v in variants:
    t0 = time.time()
    s = pkg.Solver(algo, G.n, G.row_ptr, G.col, device=0, **v)
    b = time.time() - t0
    s.run(q)
    info = s.run(q)
    st = s.stats()
    print(json.dumps(dict(variant=v, algo=algo, us_per_iter=round(info["us_per_iter"], 1), iters=info["iterations"],
                          pred=round(info["predicted_us_per_iter"], 1), two_phase=st["two_phase"],
                          groups=st["pb_groups"], chunks=st["pb_chunks"], bins=st["pb_bins"], long=st["pb_long_bins"],
                          build_s=round(b, 1))), flush=True)
    s.close()
