"""c4 (it-2004-shaped, 1.15 B edges) on one B200: the auto-tuner with the beyond-L2 x regime
(reading R32) against manual tilings, predicted vs measured, valued SpMV and PageRank.
Usage (GPU box): python bench/experiment_c4_model.py > gpurun_out/c4_model.jsonl"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import graphgen  # noqa: E402
from paper_1103_2405_b200 import Plan, Solver  # noqa: E402


def out(**kw):
    print(json.dumps(kw), flush=True)


t0 = time.time()
G = graphgen.make_graph("c4")
out(step="generate", n=G.n, m=G.m, gen_s=round(time.time() - t0, 1))
val = graphgen.edge_values(G.keys)
x = graphgen.uniform_f32(G.n, seed=3)
xt = torch.from_numpy(x).cuda()
yt = torch.empty(G.n, device="cuda")
variants = json.loads(os.environ.get("VARIANTS", "null")) or [
    dict(), dict(tile_width=49152, num_tiles=16),
    dict(tile_width=1 << 22, num_tiles=1, stage_x=0), dict(tile_width=1 << 23, num_tiles=4, stage_x=0),
    dict(tile_width=1 << 22, num_tiles=4, stage_x=0), dict(tile_width=1 << 21, num_tiles=2, stage_x=0)]
y_ref = None
for v in variants:
    t1 = time.time()
    pl = Plan(G.n, G.n, G.row_ptr, G.col, val, device=0, workload_size=1024, **v) if v else \
        Plan(G.n, G.n, G.row_ptr, G.col, val, device=0)
    b_s = time.time() - t1
    for _ in range(3):
        pl.execute(xt, yt)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        pl.execute(xt, yt)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1000 / 20
    y = yt.cpu().numpy()
    if y_ref is None:
        y_ref = y
    st = pl.stats()
    out(step="spmv_valued", opt=v or "auto", us=round(us, 1), predicted_us=round(st["predicted_us"], 1),
        gflops=round(2 * G.m / us / 1e3, 1), build_s=round(b_s, 1),
        max_rel_dev_vs_first=float(np.max(np.abs(y - y_ref) / (np.abs(y_ref) + 1e-30))),
        plan=dict(num_tiles=st["num_tiles"], tile_width=st["tile_width"], tile_staged=st["tile_staged"]))
    pl.close()
    torch.cuda.empty_cache()
del xt, yt, val
t1 = time.time()
s = Solver("pagerank", G.n, G.row_ptr, G.col, device=0)
b_s = time.time() - t1
s.run()
info = s.run()
st = s.stats()
out(step="pagerank", build_s=round(b_s, 1), iterations=info["iterations"], us_per_iter=round(info["us_per_iter"], 1),
    iters_per_s=round(1e6 / info["us_per_iter"], 1), predicted_us_per_iter=round(info["predicted_us_per_iter"], 1),
    plan=dict(num_tiles=st["num_tiles"], tile_width=st["tile_width"], tile_staged=st["tile_staged"]))
