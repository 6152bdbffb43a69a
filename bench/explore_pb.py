"""Two-phase tiles on a config: time spmv_execute (CUDA events) over parameter variants and check
sampled rows against an fp64 recomputation.  Usage: python bench/explore_pb.py c2 [json variants]"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import graphgen  # noqa: E402
import paper_1103_2405_b200 as pkg  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
variants = json.loads(sys.argv[2]) if len(sys.argv) > 2 else [dict(two_phase=0), dict(two_phase=1)]
pattern = os.environ.get("PATTERN", "0") == "1"
t0 = time.time()
G = graphgen.make_graph(cfg)
val = None if pattern else graphgen.edge_values(G.keys, seed=graphgen.SEED_VAL, mode=1)
x = graphgen.uniform_f32(G.n, seed=graphgen.SEED_X)
print(json.dumps(dict(cfg=cfg, n=G.n, m=G.m, gen_s=round(time.time() - t0, 1))), flush=True)
xt = torch.from_numpy(x).cuda()
yt = torch.empty(G.n, device="cuda")
rng = np.random.default_rng(0)
rows = rng.choice(G.n, 3000, replace=False)
lens = np.diff(G.row_ptr)
rows = np.unique(np.concatenate([rows, np.argsort(lens)[-20:]]))
def _v(r):
    a, b = G.row_ptr[r], G.row_ptr[r + 1]
    return val[a:b].astype(np.float64) if val is not None else np.ones(b - a)
ref = np.array([np.dot(_v(r), x[G.col[G.row_ptr[r]:G.row_ptr[r + 1]]].astype(np.float64)) for r in rows])
bnd = np.array([np.sum(np.abs(_v(r) * x[G.col[G.row_ptr[r]:G.row_ptr[r + 1]]])) for r in rows])
for v in variants:
    t1 = time.time()
    p = pkg.Plan(G.n, G.n, G.row_ptr, G.col, val, device=0, **v)
    build = time.time() - t1
    st = p.stats()
    for _ in range(5):
        p.execute(xt, yt)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 50
    e0.record()
    for _ in range(reps):
        p.execute(xt, yt)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / reps * 1e3
    y = yt.cpu().numpy()
    err = np.abs(y[rows].astype(np.float64) - ref)
    ok = bool((err <= 1e-5 * bnd + 1e-30).all())
    out = dict(variant=v, us=round(us, 2), gflops=round(2 * G.m / us / 1e3, 1),
               alg_GBps=round(((4 if pattern else 8) * G.m + 12 * G.n) / us / 1e3, 1), parity=ok,
               build_s=round(build, 2), two_phase=st["two_phase"], pred_tp=round(st["two_phase_predicted_us"], 1),
               pred_op=round(st["one_pass_predicted_us"], 1), groups=st["pb_groups"], chunks=st["pb_chunks"],
               bins=st["pb_bins"], long=st["pb_long_bins"], resident_warps=st["resident_warps"],
               dev_MB=round(st["device_bytes"] / 1e6, 1))
    print(json.dumps(out), flush=True)
    del p
