"""Exploration harness (not the bench contract): time spmv_execute on one config under several
environment settings read at plan creation (TCSPMV_PREFIX, TCSPMV_L1_HOT, ...), for the library
TCSPMV_LIB points at.  The graph is cached under /tmp between processes of one gpurun call.
Usage: ENVS='[{"TCSPMV_PREFIX": "49152"}, {}]' python bench/explore_env.py c2 [--pattern]"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import graphgen  # noqa: E402
from paper_1103_2405_b200 import Plan  # noqa: E402


def load(cfg):
    path = f"/tmp/tcspmv_{cfg}.npz"
    if os.path.exists(path):
        z = np.load(path)
        return int(z["n"]), z["rp"], z["col"], z["val"]
    G = graphgen.make_graph(cfg)
    val = graphgen.edge_values(G.keys)
    np.savez(path, n=G.n, rp=G.row_ptr, col=G.col, val=val)
    return G.n, G.row_ptr, G.col, val


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
    pattern = "--pattern" in sys.argv
    n, rp, col, val = load(cfg)
    m = len(col)
    if pattern:
        val = None
    x = graphgen.uniform_f32(n, seed=3)
    xt = torch.from_numpy(x).cuda()
    yt = torch.empty(n, device="cuda")
    opt = json.loads(os.environ.get("OPT", '{"num_tiles": 0, "workload_size": 1024}'))
    lib = os.path.basename(os.environ.get("TCSPMV_LIB", "libtcspmv.so"))
    y0 = None
    base_env = dict(os.environ)
    for env in json.loads(os.environ.get("ENVS", "[{}]")):
        for k in ("TCSPMV_PREFIX", "TCSPMV_L1_HOT", "TCSPMV_CARVEOUT"):
            os.environ.pop(k, None)
            if k in base_env:
                os.environ[k] = base_env[k]
        os.environ.update({k: str(v) for k, v in env.items()})
        p = Plan(n, n, rp, col, val, device=0, **opt)
        for _ in range(5):
            p.execute(xt, yt)
        torch.cuda.synchronize()
        res = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(50):
                p.execute(xt, yt)
            e1.record()
            torch.cuda.synchronize()
            res.append(e0.elapsed_time(e1) * 1000 / 50)
        us = float(np.median(res))
        y = yt.cpu().numpy()
        if y0 is None:
            y0 = y
        dev = float(np.max(np.abs(y - y0)))
        print(json.dumps(dict(lib=lib, cfg=cfg, pattern=pattern, env=env, us=round(us, 1),
                              gflops=round(2 * m / us / 1e3, 1), maxdev_vs_first=dev)), flush=True)
        p.close()


if __name__ == "__main__":
    main()
