"""Exploration harness (not the bench contract): time spmv_execute on a config under several
plan options.  Usage: python bench/explore_spmv.py c2 [--pattern]"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import graphgen  # noqa: E402
from paper_1103_2405_b200 import Plan  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
    pattern = "--pattern" in sys.argv
    t0 = time.time()
    G = graphgen.make_graph(cfg)
    rp, col = G.row_ptr, G.col
    val = None if pattern else graphgen.edge_values(G.keys)
    x = graphgen.uniform_f32(G.n, seed=3)
    print(json.dumps(dict(cfg=cfg, n=G.n, m=G.m, gen_s=round(time.time() - t0, 1))), flush=True)
    xt = torch.from_numpy(x).cuda()
    yt = torch.empty(G.n, device="cuda")
    variants = json.loads(os.environ.get("VARIANTS", "null")) or [
        dict(num_tiles=0, workload_size=1024),
        dict(tile_width=49152, num_tiles=1, workload_size=1024),
        dict(tile_width=49152, num_tiles=1, workload_size=1024, stage_x=0),
        dict(tile_width=49152, num_tiles=3, workload_size=1024),
        dict(tile_width=49152, num_tiles=3, workload_size=1024, stage_x=0),
        dict(tile_width=24576, num_tiles=4, workload_size=1024),
        dict(tile_width=49152, num_tiles=6, workload_size=1024),
        dict(tile_width=49152, num_tiles=10, workload_size=1024),
        dict(tile_width=49152, num_tiles=10, workload_size=1024, stage_x=0),
        dict(tile_width=49152, num_tiles=16, workload_size=1024),
        dict(tile_width=49152, num_tiles=3, workload_size=256),
        dict(tile_width=49152, num_tiles=3, workload_size=4096),
    ]
    for v in variants:
        t0 = time.time()
        p = Plan(G.n, G.n, rp, col, val, device=0, **v)
        build_s = time.time() - t0
        st = p.stats()
        for _ in range(3):
            p.execute(xt, yt)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 20
        e0.record()
        for _ in range(reps):
            p.execute(xt, yt)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1000 / reps
        bytes_alg = (4 if pattern else 8) * G.m + 12 * G.n
        print(json.dumps(dict(opt=v, us=round(us, 1), gflops=round(2 * G.m / us / 1e3, 1),
                              alg_GBps=round(bytes_alg / us / 1e3, 1), build_s=round(build_s, 1),
                              launches=p.launches, slots_per_nnz=round(st["n_slots"] / G.m, 3),
                              tile_nnz=st["tile_nnz"], wl=st["wl"], staged=st["tile_staged"])), flush=True)
        p.close()


if __name__ == "__main__":
    main()
