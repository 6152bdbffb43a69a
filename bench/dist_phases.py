"""Row-partitioned PageRank through the loopback transport (P logical ranks on ONE GPU, one host
thread each): iterations/s and the per-phase split (local SpMV with fused epilogue, exchange,
partial sums) per P.  The ranks share the device, so this shows the protocol's structure and
costs, not multi-GPU scaling.  Usage: python bench/dist_phases.py c2 [P ...] [--exchange 1]"""
import json
import os
import sys
import threading
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import graphgen  # noqa: E402
import paper_1103_2405_b200 as pkg  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
cfg = args[0] if args else "c2"
Ps = [int(a) for a in args[1:]] or [1, 2, 4, 8]
ex = 1 if "--exchange" in sys.argv else 0
algo = os.environ.get("ALGO", "pagerank")
t0 = time.time()
G = graphgen.make_graph(cfg)
gen = time.time() - t0
for P in Ps:
    comms = pkg.Comm.loopback(P, 0)
    out = [None] * P
    builds = [0.0] * P

    def body(r):
        tb = time.time()
        s = pkg.Solver(algo, G.n, G.row_ptr, G.col, device=0, comm=comms[r], iter_kw=dict(exchange=ex))
        builds[r] = time.time() - tb
        s.run(0, stream=0)
        out[r] = s.run(0, stream=0)
        s.close()

    th = [threading.Thread(target=body, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for c in comms:
        c.close()
    worst = max(out, key=lambda i: i["ms_total"])
    ph = np.max(np.array([o["phase_us"] for o in out]), axis=0)
    print(json.dumps(dict(cfg=cfg, algo=algo, P=P, exchange=ex, iterations=worst["iterations"],
                          us_per_iter=round(worst["us_per_iter"], 1),
                          iters_per_s=round(1e6 / worst["us_per_iter"], 1),
                          phase_us_max_over_ranks={"spmv": round(ph[0], 1), "exchange": round(ph[1], 1),
                                                   "rest": round(ph[2], 1)},
                          build_s=round(max(builds), 1), gen_s=round(gen, 1),
                          note="loopback: P logical ranks share one GPU")), flush=True)
