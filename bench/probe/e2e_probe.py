"""e2e pipeline probe: spmv_execute_host_batch on c2 for several batch counts and buffer depths."""
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import graphgen  # noqa: E402
import paper_1103_2405_b200 as pkg  # noqa: E402

G = graphgen.make_graph("c2")
val = graphgen.edge_values(G.keys)
x = graphgen.uniform_f32(G.n, seed=3)
plan = pkg.Plan(G.n, G.n, G.row_ptr, G.col, val, device=0)
streams = {"default": torch.cuda.current_stream(), "side": torch.cuda.Stream()}
for (sname, stream), cnt in [(kv, c) for kv in streams.items() for c in (32,)]:
    xh = torch.from_numpy(x).unsqueeze(0).expand(cnt, G.n).contiguous().pin_memory()
    yh = torch.empty((cnt, G.n), dtype=torch.float32).pin_memory()
    for pipe in ("3",):
        os.environ["TCSPMV_PIPE"] = pipe
        call = lambda c: pkg._capi.check(pkg.lib().spmv_execute_host_batch(
            plan._h, ctypes.c_void_p(xh.data_ptr()), ctypes.c_void_p(yh.data_ptr()), c,
            ctypes.c_void_p(stream.cuda_stream)), "e2e")
        call(3)
        res = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            call(cnt)
            e1.record(stream)
            torch.cuda.synchronize()
            res.append(e0.elapsed_time(e1) / cnt)
        print(json.dumps(dict(stream=sname, count=cnt, pipe=int(pipe), ms_per_step=[round(r, 4) for r in res])), flush=True)
