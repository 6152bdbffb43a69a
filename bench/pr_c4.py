"""c4 PageRank, single-GPU solver (multi-tile plan): us per iteration (device generator input)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import graphgen  # noqa: E402
from paper_1103_2405_b200 import Solver  # noqa: E402

dg = graphgen.DeviceGraph("c4")
G = graphgen.graph_from_keys("c4", dg.n, dg.keys())
dg.close()
s = Solver("pagerank", G.n, G.row_ptr, G.col, device=0)
s.run()
info = s.run()
print(json.dumps(dict(lib=os.path.basename(os.environ.get("TCSPMV_LIB", "libtcspmv.so")), c4_us_per_iter=round(info["us_per_iter"], 1),
                      it=info["iterations"], tiles=s.stats()["num_tiles"])), flush=True)
