"""Workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck): one-pass SpMV
(single tile, staged multi-tile, paper mode), two-phase SpMV, and the PageRank / HITS / RWR
epilogue kernels through the row-partitioned solver at world 1 (a host-driven loop: the
single-GPU solvers run inside a CUDA graph with a WHILE node, which the sanitizer tools do not
instrument), the slices transport at 3 ranks and batched RWR's host-driven loop.  The multi-tile
one-pass plan is chained by programmatic dependent launch.  Usage: python bench/sanitize_run.py [c1|t_small]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import graphgen  # noqa: E402
import paper_1103_2405_b200 as pkg  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c1"
G = graphgen.make_graph(cfg)
val = graphgen.edge_values(G.keys, seed=graphgen.SEED_VAL, mode=1)
x = torch.from_numpy(graphgen.uniform_f32(G.n, seed=graphgen.SEED_X)).cuda()
y = torch.empty(G.n, device="cuda")
for opt in (dict(two_phase=0), dict(two_phase=0, tile_width=4096, num_tiles=3, workload_size=256),
            dict(two_phase=0, num_tiles=0, split_long_rows=0, align_rm=32),
            dict(two_phase=1), dict(two_phase=1, pb_region=512, pb_chunk=600, pb_group=50000)):
    p = pkg.Plan(G.n, G.n, G.row_ptr, G.col, val, device=0, **opt)
    for _ in range(2):
        p.execute(x, y)
    torch.cuda.synchronize()
    print(cfg, opt, float(y.sum()), flush=True)
    p.close()
q = int(np.nonzero(np.diff(G.row_ptr) > 0)[0][0])
comm = pkg.Comm(0, 1, b"\0" * 128, 0)
for algo in ("pagerank", "hits", "rwr"):
    for ex in (0, 1):
        s = pkg.Solver(algo, G.n, G.row_ptr, G.col, device=0, comm=comm, iter_kw=dict(fixed_iters=3, exchange=ex))
        info = s.run(q, stream=0)
        s.result()
        print(cfg, algo, "exchange", ex, info["iterations"], flush=True)
        s.close()
comm.close()
# round 2: the slices transport (3 row slices of one solver sharing one exchange buffer, one host
# thread each) and batched RWR through its host-driven loop
import threading  # noqa: E402
for algo in ("pagerank", "hits"):
    comms = pkg.Comm.slices(3, 0)
    outs = [None] * 3

    def body(r):
        s = pkg.Solver(algo, G.n, G.row_ptr, G.col, device=0, comm=comms[r], iter_kw=dict(fixed_iters=3))
        outs[r] = s.run(0, stream=0)["iterations"]
        s.result()
        s.close()
    th = [threading.Thread(target=body, args=(r,)) for r in range(3)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for c in comms:
        c.close()
    print(cfg, algo, "slices", outs, flush=True)
s = pkg.Solver("rwr", G.n, G.row_ptr, G.col, device=0, iter_kw=dict(fixed_iters=3, host_loop=1))
deg = np.diff(G.row_ptr) + np.bincount(G.col, minlength=G.n)
qs = np.nonzero(deg > 0)[0][:25]
print(cfg, "rwr batch", s.run_batch(qs)["iterations"], flush=True)
s.close()
print("done")
