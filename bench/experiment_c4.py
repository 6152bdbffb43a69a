"""BASELINE configs[3] on one B200: it-2004-shaped web graph (Graph500 R-MAT scale 26, n =
41,291,594, m = 1,150,725,436).  Every measurement is printed as its own JSON line as soon as it
is done (a timeout keeps what finished):
  1. PageRank to 1e-6 with the auto-tuned plan: iterations, us/iteration, iterations/s, GFLOP/s;
  2. full-size parity: the fp64 oracle run for the same iteration count, L1 distance and sum(p)
     (R14), with the oracle's time per iteration on the host cores (cpu baseline);
  3. valued SpMV (y = A x) with the auto plan and L2-sized hub tiles (x = 165 MB > the 126 MB L2,
     so here tiling decides whether the hub gathers stay on chip: Solution 1 at the L2 level);
  4. HITS on the 2n-row block matrix (c5's algorithm at c4 scale) when C4_HITS=1.
Usage (GPU box): python bench/experiment_c4.py > gpurun_out/c4.jsonl"""
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


def plan_info(st):
    return dict(num_tiles=st["num_tiles"], tile_width=st["tile_width"], wl=st["wl"],
                tile_staged=st["tile_staged"], predicted_us=round(st["predicted_us"], 1),
                device_bytes=st["device_bytes"], build_ms=round(st["build_ms"], 1))


t0 = time.time()
G = graphgen.make_graph("c4")
deg_out = np.diff(G.row_ptr)
out(step="generate", config="c4 it-2004-shaped R-MAT s26 Graph500", n=G.n, m=G.m,
    gen_s=round(time.time() - t0, 1), dangling_frac=round(float((deg_out == 0).mean()), 4),
    max_in_degree=int(np.bincount(G.col, minlength=G.n).max()))

# 1. PageRank (pattern A^T, fused Eq. 6 epilogue, device-side loop)
t0 = time.time()
s = Solver("pagerank", G.n, G.row_ptr, G.col, device=0)
build_s = time.time() - t0
s.run()
info = s.run()
p = s.result()
out(step="pagerank", build_s=round(build_s, 1), iterations=info["iterations"],
    converged=info["converged"], us_per_iter=round(info["us_per_iter"], 1),
    iters_per_s=round(1e6 / info["us_per_iter"], 1),
    gflops=round(2 * G.m / info["us_per_iter"] / 1e3, 1),
    alg_GBps=round((4 * G.m + 12 * G.n + 20 * G.n) / info["us_per_iter"] / 1e3, 1),
    predicted_us_per_iter=round(info["predicted_us_per_iter"], 1), plan=plan_info(s.stats()))
s.close()
torch.cuda.empty_cache()

# 2. full-size parity against the oracle (same iteration count) + oracle timing
if os.environ.get("C4_ORACLE", "1") == "1":
    import oracle
    t0 = time.perf_counter()
    pr, r = oracle.pagerank(G.n, G.row_ptr, G.col, fixed_iters=info["iterations"])
    dt = time.perf_counter() - t0
    out(step="pagerank_parity", oracle_iterations=r.iterations, l1=float(np.abs(p - pr).sum()),
        sum_p=float(p.astype(np.float64).sum()), oracle_s=round(dt, 1),
        oracle_s_per_iter=round(dt / max(r.iterations, 1), 2),
        cores=len(os.sched_getaffinity(0)), bound="1e-6 L1 (north_star)")
    del pr

# 3. valued SpMV: auto plan vs L2-sized hub tiles
val = graphgen.edge_values(G.keys)
x = graphgen.uniform_f32(G.n, seed=3)
xt = torch.from_numpy(x).cuda()
yt = torch.empty(G.n, device="cuda")
variants = [dict()] + [dict(tile_width=tw, num_tiles=1, stage_x=0, workload_size=1024)
                       for tw in (4 << 20, 8 << 20, 16 << 20)]
y_ref = None
for v in variants:
    t0 = time.time()
    pl = Plan(G.n, G.n, G.row_ptr, G.col, val, device=0, **v)
    b_s = time.time() - t0
    for _ in range(3):
        pl.execute(xt, yt)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record()
    for _ in range(reps):
        pl.execute(xt, yt)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1000 / reps
    y = yt.cpu().numpy()
    if y_ref is None:
        # sampled full-size parity: 4096 rows against the oracle's definition (O1)
        rng = np.random.default_rng(11)
        rows = np.sort(rng.choice(G.n, 4096, replace=False))
        import oracle
        sub_rp = np.concatenate([[0], np.cumsum(deg_out[rows])]).astype(np.int64)
        idx = np.concatenate([np.arange(G.row_ptr[r], G.row_ptr[r + 1]) for r in rows])
        yo, bo = oracle.spmv(sub_rp, G.col[idx], val[idx], x)
        ok = bool(np.all(np.abs(y[rows] - yo) <= 1e-5 * bo + 1e-30))
        y_ref = y
        out(step="spmv_parity_sampled", rows=4096, all_within_tol=ok,
            max_rel=float(np.max(np.abs(y[rows] - yo) / (bo + 1e-30))))
    out(step="spmv_valued", opt=v, us=round(us, 1), gflops=round(2 * G.m / us / 1e3, 1),
        alg_GBps=round((8 * G.m + 12 * G.n) / us / 1e3, 1), build_s=round(b_s, 1),
        max_dev_vs_auto=float(np.max(np.abs(y - y_ref))), plan=plan_info(pl.stats()))
    pl.close()
    torch.cuda.empty_cache()
del val, xt, yt

# 4. HITS on the block matrix (2n rows, 2m entries)
if os.environ.get("C4_HITS", "0") == "1":
    t0 = time.time()
    s = Solver("hits", G.n, G.row_ptr, G.col, device=0)
    build_s = time.time() - t0
    s.run()
    info = s.run()
    out(step="hits", build_s=round(build_s, 1), iterations=info["iterations"],
        us_per_iter=round(info["us_per_iter"], 1), iters_per_s=round(1e6 / info["us_per_iter"], 1),
        gflops=round(4 * G.m / info["us_per_iter"] / 1e3, 1), plan=plan_info(s.stats()))
    s.close()
