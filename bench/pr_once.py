"""PageRank on c2 for a few fixed iterations with the host-driven loop (kernels visible to ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import graphgen  # noqa: E402
from paper_1103_2405_b200 import Solver  # noqa: E402

G = graphgen.make_graph(sys.argv[1] if len(sys.argv) > 1 else "c2")
s = Solver("pagerank", G.n, G.row_ptr, G.col, device=0, iter_kw=dict(fixed_iters=4, host_loop=1))
print(s.run(), s.stats()["wl"], flush=True)
