"""One plan, a few launches (for ncu captures of the two-phase kernel)."""
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import graphgen
import paper_1103_2405_b200 as pkg
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
opt = json.loads(sys.argv[2]) if len(sys.argv) > 2 else dict(two_phase=1)
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
pattern = os.environ.get("PATTERN", "0") == "1"
G = graphgen.make_graph(cfg)
val = None if pattern else graphgen.edge_values(G.keys, seed=graphgen.SEED_VAL, mode=1)
x = graphgen.uniform_f32(G.n, seed=graphgen.SEED_X)
p = pkg.Plan(G.n, G.n, G.row_ptr, G.col, val, device=0, **opt)
xt = torch.from_numpy(x).cuda(); yt = torch.empty(G.n, device="cuda")
for _ in range(reps):
    p.execute(xt, yt)
torch.cuda.synchronize()
print(json.dumps(p.stats()["two_phase"]))
