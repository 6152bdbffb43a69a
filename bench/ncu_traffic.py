"""Helper of bench.py (run under ncu): build the bench plan on the c2 workload and launch it three
times, so that one launch can be captured for its DRAM bytes."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import graphgen  # noqa: E402
import paper_1103_2405_b200 as pkg  # noqa: E402

G = graphgen.make_graph("c2")
val = graphgen.edge_values(G.keys, seed=graphgen.SEED_VAL, mode=1)
x = torch.from_numpy(graphgen.uniform_f32(G.n, seed=graphgen.SEED_X)).cuda()
y = torch.empty(G.n, device="cuda")
p = pkg.Plan(G.n, G.n, G.row_ptr, G.col, val, device=0)
for _ in range(3):
    p.execute(x, y)
torch.cuda.synchronize()
print(float(np.float64(y.sum().item())))
