"""§8(f) f4 (Appendix D): SpMV off the power-law regime -- dense and
FEM-like banded matrices, where x gathers are sequential and the kernel should approach the HBM
roofline.  Auto-tuned plans; reports us, GFLOP/s, algorithmic GB/s (8 B per entry + 12 B per row)
and the fraction of the measured copy peak.
Usage (GPU box): python bench/experiment_f4.py > profiles/r01_f4_dense_banded.json"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import graphgen  # noqa: E402
from paper_1103_2405_b200 import Plan  # noqa: E402


def peak():
    try:
        d = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                        "MEASURED_PEAKS.json")))
        for k in ("hbm_gbs",):
            if k in d:
                return float(d[k])
    except Exception:
        pass
    return 6446.3


def run(name, nr, nc, rp, col, val, reps=50):
    p = Plan(nr, nc, rp, col, val, device=0)
    st = p.stats()
    x = torch.from_numpy(graphgen.uniform_f32(nc, seed=graphgen.SEED_X)).cuda()
    y = torch.empty(nr, device="cuda")
    for _ in range(5):
        p.execute(x, y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        p.execute(x, y)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / reps
    m = len(col)
    gbs = (8.0 * m + 12.0 * nr) / us / 1e3
    rec = dict(matrix=name, n_rows=nr, n_cols=nc, nnz=m, us=round(us, 2), gflops=round(2 * m / us / 1e3, 1),
               alg_GBps=round(gbs, 1), frac_of_copy_peak=round(gbs / peak(), 3),
               plan=dict(num_tiles=st["num_tiles"], wl=st["wl"], predicted_us=round(st["predicted_us"], 1)))
    print(json.dumps(rec), flush=True)
    p.close()
    return rec


def main():
    out = []
    for nr, nc in ((2048, 2048), (8192, 8192), (16384, 16384)):
        rp, col, val = graphgen.dense_csr(nr, nc)
        out.append(run(f"dense_{nr}x{nc}", nr, nc, rp, col, val))
    for n, hb, drop in ((4_000_000, 13, 0.0), (4_000_000, 13, 0.4), (1_000_000, 60, 0.0)):
        rp, col, val = graphgen.banded_csr(n, hb, drop=drop)
        out.append(run(f"banded_n{n}_hb{hb}_drop{drop}", n, n, rp, col, val))
    json.dump(out, sys.stderr)


if __name__ == "__main__":
    main()
