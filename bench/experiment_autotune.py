"""BASELINE configs[2] (Sec. 4.4, Fig. 5): on Flickr/YouTube-shaped capped
Chung-Lu graphs over the power-law exponent sweep, compare the auto-tuned plan (Alg. 1-3 with the
measured offline table) against an exhaustive search over tile count and workload size, and the
model's predicted time against the measured time.

The one-pass tiles are tuned (two_phase = 0: Alg. 1-3 is the paper's tuner); the two-phase time
is reported beside it.  --c2 adds the LiveJournal-shaped graph.
Usage (GPU box): python bench/experiment_autotune.py [--quick] [--c2] > profiles/r02_autotune.json
"""
import ctypes
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import graphgen  # noqa: E402
import paper_1103_2405_b200 as pkg  # noqa: E402


def time_plan(p, xt, yt, reps=20):
    for _ in range(3):
        p.execute(xt, yt)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        p.execute(xt, yt)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1000 / reps


def main():
    quick = "--quick" in sys.argv
    alphas = [1.8, 2.2, 2.6] if quick else [1.8, 2.0, 2.2, 2.4, 2.6]
    shapes = {"flickr": (1_700_000, 22_600_000), "youtube": (1_100_000, 4_900_000)}
    if "--graph" in sys.argv:
        g = sys.argv[sys.argv.index("--graph") + 1]
        shapes = {g: shapes[g]}
    tile_counts = (0,) if "--t0" in sys.argv else (0, 1, 2, 4)
    out = []
    cases = [(name, n, m, a) for name, (n, m) in shapes.items() for a in alphas]
    if "--c2" in sys.argv:
        cases.insert(0, ("c2", None, None, None))
    for name, n, m, a in cases:
        if True:
            if name == "c2":
                G = graphgen.make_graph("c2")
                n = G.n
            else:
                keys = graphgen.chung_lu_edges(n, m, a, 2e4)
                G = graphgen.graph_from_keys(f"{name}_a{a}", n, keys)
            val = graphgen.edge_values(G.keys)
            x = graphgen.uniform_f32(n, seed=graphgen.SEED_X)
            xt = torch.from_numpy(x).cuda()
            yt = torch.empty(n, device="cuda")
            auto = pkg.Plan(n, n, G.row_ptr, G.col, val, device=0, two_phase=0)
            st = auto.stats()
            auto_us = time_plan(auto, xt, yt)
            auto_launch = st["predicted_us"]
            auto.close()
            tp = pkg.Plan(n, n, G.row_ptr, G.col, val, device=0, two_phase=1)
            tp_us, tp_pred = time_plan(tp, xt, yt), tp.stats()["two_phase_predicted_us"]
            tp.close()
            best = None
            grid = []
            for tw in (24576, 49152):
                for T in tile_counts:
                    if T == 0 and tw != 24576:
                        continue
                    for wl in (256, 512, 1024, 2048, 4096, 8192):
                        p = pkg.Plan(n, n, G.row_ptr, G.col, val, device=0, tile_width=tw, num_tiles=T,
                                     workload_size=wl, two_phase=0)
                        s2 = p.stats()
                        us = time_plan(p, xt, yt)
                        grid.append(dict(tile_width=tw, num_tiles=s2["num_tiles"], wl=wl, us=round(us, 2),
                                         predicted_us=round(s2["predicted_us"], 2)))
                        if best is None or us < best["us"]:
                            best = grid[-1]
                        p.close()
            rec = dict(graph=name, alpha=a, n=n, m=G.m,
                       auto=dict(num_tiles=st["num_tiles"], tile_width=st["tile_width"], wl=st["wl"],
                                 us=round(auto_us, 2), predicted_us=round(auto_launch, 2),
                                 composite_threshold=st["composite_threshold"]),
                       exhaustive_best=best,
                       auto_vs_best=round(best["us"] / auto_us, 4),
                       prediction_error=round(abs(auto_launch - auto_us) / auto_us, 4),
                       two_phase=dict(us=round(tp_us, 2), predicted_us=round(tp_pred, 2)),
                       grid=grid)
            out.append(rec)
            print(json.dumps({k: rec[k] for k in ("graph", "alpha", "auto", "exhaustive_best", "auto_vs_best",
                                                  "prediction_error", "two_phase")}), file=sys.stderr, flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
