"""L2-level tiling on c4 (x = 165 MB > the 126 MB L2): pattern SpMV on the PageRank matrix A^T
(the per-iteration product of bench/experiment_c4.py) for tile widths whose x segment fits L2,
unstaged (gathers through L1/L2), against the auto-tuned plan.  One JSON line per plan.
Usage (GPU box): python bench/experiment_c4_tiles.py > gpurun_out/c4_tiles.jsonl"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import graphgen  # noqa: E402
from paper_1103_2405_b200 import Plan, Solver  # noqa: E402

t0 = time.time()
G = graphgen.make_graph(os.environ.get("CFG", "c4"))
rpT, colT = graphgen.keys_to_csr(G.keys, G.n, transpose=True)
n, m = G.n, G.m
print(json.dumps(dict(step="generate", n=n, m=m, gen_s=round(time.time() - t0, 1))), flush=True)
x = graphgen.uniform_f32(n, seed=3)
xt = torch.from_numpy(x).cuda()
yt = torch.empty(n, device="cuda")
variants = json.loads(os.environ.get("VARIANTS", "null")) or (
    [dict()] + [dict(tile_width=tw << 20, num_tiles=int(-(-n // (tw << 20))) - 1, stage_x=0, workload_size=1024)
                for tw in (2, 4, 8, 12, 16, 24)] +
    [dict(tile_width=tw << 20, num_tiles=1, stage_x=0, workload_size=1024) for tw in (2, 4)])
best = None
for v in variants:
    t0 = time.time()
    p = Plan(n, n, rpT, colT, None, device=0, **v)
    b_s = time.time() - t0
    for _ in range(3):
        p.execute(xt, yt)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        p.execute(xt, yt)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 100
    st = p.stats()
    print(json.dumps(dict(step="spmv_pattern_AT", opt=v, us=round(us, 1), gflops=round(2 * m / us / 1e3, 1),
                          alg_GBps=round((4 * m + 12 * n) / us / 1e3, 1), build_s=round(b_s, 1),
                          num_tiles=st["num_tiles"], tile_width=st["tile_width"],
                          predicted_us=round(st["predicted_us"], 1),
                          tile_nnz=st["tile_nnz"][: st["num_tiles"] + 1],
                          tile_us_pred=[round(u, 1) for u in st["tile_predicted_us"][: st["num_tiles"] + 1]])),
          flush=True)
    if best is None or us < best[0]:
        best = (us, v)
    p.close()
    torch.cuda.empty_cache()
if os.environ.get("C4_PR", "1") == "1" and best[1]:
    s = Solver("pagerank", n, G.row_ptr, G.col, device=0, **best[1])
    s.run()
    info = s.run()
    print(json.dumps(dict(step="pagerank_best_tiling", opt=best[1], iterations=info["iterations"],
                          us_per_iter=round(info["us_per_iter"], 1),
                          iters_per_s=round(1e6 / info["us_per_iter"], 1))), flush=True)
