"""BASELINE configs[3] on one B200: it-2004-shaped web graph (Graph500 R-MAT scale 26, n =
41,291,594, m = 1,150,725,436): PageRank to 1e-6 with the auto-tuned plan; reports build time,
iterations, us/iteration, iterations/s and GFLOP/s (2 m per iteration).
Usage (GPU box): python bench/experiment_c4.py > profiles/r01_c4_pagerank.json"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import graphgen  # noqa: E402
from paper_1103_2405_b200 import Solver  # noqa: E402

t0 = time.time()
G = graphgen.make_graph("c4")
gen_s = time.time() - t0
t0 = time.time()
s = Solver("pagerank", G.n, G.row_ptr, G.col, device=0)
build_s = time.time() - t0
s.run()
info = s.run()
st = s.stats()
print(json.dumps(dict(config="c4 it-2004-shaped R-MAT s26", n=G.n, m=G.m, gen_s=round(gen_s, 1),
                      build_s=round(build_s, 1), iterations=info["iterations"],
                      us_per_iter=round(info["us_per_iter"], 1),
                      iters_per_s=round(1e6 / info["us_per_iter"], 1),
                      gflops=round(2 * G.m / info["us_per_iter"] / 1e3, 1),
                      plan=dict(num_tiles=st["num_tiles"], tile_width=st["tile_width"], wl=st["wl"],
                                predicted_us=round(st["predicted_us"], 1), device_bytes=st["device_bytes"]))))
