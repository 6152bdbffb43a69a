"""c4 (1.15 B entries) valued SpMV with the auto plan, executed a few times, for an ncu capture of
its tile launches (bench/runs/run74.sh)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import graphgen  # noqa: E402
from paper_1103_2405_b200 import Plan  # noqa: E402

G = graphgen.make_graph("c4")
val = graphgen.edge_values(G.keys)
x = torch.from_numpy(graphgen.uniform_f32(G.n, seed=3)).cuda()
y = torch.empty(G.n, device="cuda")
p = Plan(G.n, G.n, G.row_ptr, G.col, val, device=0)
print(p.stats()["num_tiles"], p.stats()["tile_width"], flush=True)
for _ in range(3):
    p.execute(x, y)
torch.cuda.synchronize()
