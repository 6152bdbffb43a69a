"""§8(f) f2: model-driven format ablations on the same kernels:
composite (Alg. 3) vs row-major only (CSR-vector) vs column-major only (ELL), untiled and tiled,
B200 mode vs the paper's parameters (WL >= longest row, align 32).  Each variant is auto-tuned by
the model within its constraints; measured and predicted us per SpMV are reported side by side.
Usage (GPU box): python bench/experiment_f2.py [c2|c3_flickr ...] > profiles/r01_f2_ablation.json"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import graphgen  # noqa: E402
from paper_1103_2405_b200 import Plan  # noqa: E402

VARIANTS = [
    ("composite", dict(num_tiles=0)),
    ("csr_vector", dict(num_tiles=0, orient=1)),
    ("ell", dict(num_tiles=0, orient=2)),
    ("composite_tiled", dict(tile_width=49152, num_tiles=2)),
    ("csr_vector_tiled", dict(tile_width=49152, num_tiles=2, orient=1)),
    ("ell_tiled", dict(tile_width=49152, num_tiles=2, orient=2)),
    ("composite_auto", dict()),
    ("paper_params", dict(split_long_rows=0, align_rm=32)),
]


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
    cfgs = [a for a in sys.argv[1:] if not a.startswith("-")] or ["c2", "c3_flickr"]
    out = []
    for cfg in cfgs:
        G = graphgen.make_graph(cfg)
        val = graphgen.edge_values(G.keys)
        xt = torch.from_numpy(graphgen.uniform_f32(G.n, seed=graphgen.SEED_X)).cuda()
        yt = torch.empty(G.n, device="cuda")
        for name, opt in VARIANTS:
            try:
                p = Plan(G.n, G.n, G.row_ptr, G.col, val, device=0, **opt)
            except Exception as e:   # e.g. paper mode on a huge longest row
                rec = dict(config=cfg, variant=name, error=str(e)[:200])
                print(json.dumps(rec), file=sys.stderr, flush=True)
                out.append(rec)
                continue
            st = p.stats()
            us = time_plan(p, xt, yt)
            rec = dict(config=cfg, variant=name, opt=opt, us=round(us, 2), gflops=round(2 * G.m / us / 1e3, 1),
                       predicted_us=round(st["predicted_us"], 2), num_tiles=st["num_tiles"], wl=st["wl"],
                       slots_per_nnz=round(st["n_slots"] / G.m, 3))
            print(json.dumps(rec), file=sys.stderr, flush=True)
            out.append(rec)
            p.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
