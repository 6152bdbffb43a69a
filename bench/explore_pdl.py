"""Programmatic dependent launch between the standalone launches of a multi-tile product (x relabel,
tile 0, tile 1, ...): CUDA-event time per product with the default library and the TC_PDL=0 build
(TCSPMV_LIB), on c2 valued with forced tilings and on the c4 auto plan (5 launches)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import graphgen  # noqa: E402
import paper_1103_2405_b200 as pkg  # noqa: E402

cases = [("c2", dict(two_phase=0, num_tiles=0)), ("c2", dict(two_phase=0, num_tiles=2, tile_width=49152)),
         ("c2", dict(two_phase=0, num_tiles=4, tile_width=49152)), ("c2", dict(two_phase=0, num_tiles=8, tile_width=16384)),
         ("c3_youtube", dict(two_phase=0, num_tiles=4, tile_width=16384))]
if os.environ.get("PDL_C4"):
    cases.append(("c4", dict(two_phase=0)))
lib = os.path.basename(os.environ.get("TCSPMV_LIB", "libtcspmv.so"))
for cfg, opt in cases:
    if cfg == "c4":
        dg = graphgen.DeviceGraph("c4")
        G = graphgen.graph_from_keys("c4", dg.n, dg.keys())
        dg.close()
    else:
        G = graphgen.make_graph(cfg)
    val = graphgen.edge_values(G.keys)
    p = pkg.Plan(G.n, G.n, G.row_ptr, G.col, val, device=0, **opt)
    x = torch.from_numpy(graphgen.uniform_f32(G.n, seed=graphgen.SEED_X)).cuda()
    y = torch.empty(G.n, device="cuda")
    reps = 20 if cfg == "c4" else 200
    for _ in range(5):
        p.execute(x, y)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        p.execute(x, y)
    e1.record()
    torch.cuda.synchronize()
    print(json.dumps(dict(lib=lib, cfg=cfg, opt=opt, launches=p.launches, us=round(e0.elapsed_time(e1) * 1e3 / reps, 2))),
          flush=True)
    p.close()
