"""Timeline of one two-phase product (spmv_pb_trace): per item kind, mean duration, reduce wait."""
import ctypes, json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import graphgen
import paper_1103_2405_b200 as pkg
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
opt = json.loads(sys.argv[2]) if len(sys.argv) > 2 else dict(two_phase=1)
pattern = os.environ.get("PATTERN", "0") == "1"
G = graphgen.make_graph(cfg)
val = None if pattern else graphgen.edge_values(G.keys, seed=graphgen.SEED_VAL, mode=1)
x = graphgen.uniform_f32(G.n, seed=graphgen.SEED_X)
p = pkg.Plan(G.n, G.n, G.row_ptr, G.col, val, device=0, **opt)
st = p.stats()
ni = st["pb_chunks"] + st["pb_bins"]
xt = torch.from_numpy(x).cuda(); yt = torch.empty(G.n, device="cuda")
for _ in range(3):
    p.execute(xt, yt)
torch.cuda.synchronize()
tr = np.zeros((ni, 4), np.int64)
s = torch.cuda.current_stream().cuda_stream
pkg._capi.check(pkg.lib().spmv_pb_trace(p._h, ctypes.c_void_p(xt.data_ptr()), ctypes.c_void_p(yt.data_ptr()),
                                        ctypes.c_void_p(s), tr.ctypes.data, ni), "trace")
t0 = tr[:, 1].min()
tr[:, 1:] -= t0
tr[tr[:, 2] < 0, 2] = 0
nch = st["pb_chunks"]
# item kinds in queue order: rebuild from the group structure is not exposed; infer: ready > 0 => reduce
red = tr[:, 2] > 0
dur = (tr[:, 3] - tr[:, 1]) / 1e3
wait = np.where(red, (tr[:, 2] - tr[:, 1]) / 1e3, 0)
span = tr[:, 3].max() / 1e3
print(json.dumps(dict(cfg=cfg, opt=opt, total_us=round(span, 1), items=int(ni), expands=int((~red).sum()), reduces=int(red.sum()),
      expand_mean_us=round(float(dur[~red].mean()), 2), expand_p90=round(float(np.percentile(dur[~red], 90)), 2),
      reduce_mean_us=round(float(dur[red].mean()), 2), reduce_p90=round(float(np.percentile(dur[red], 90)), 2),
      reduce_wait_mean_us=round(float(wait[red].mean()), 2), reduce_wait_p90=round(float(np.percentile(wait[red], 90)), 2),
      busy_frac=round(float(dur.sum() / (span * (st["resident_warps"] // 9))), 3), ctas=st["resident_warps"] // 9,
      expand_time_sum_ms=round(float(dur[~red].sum()) / 1e3, 2), reduce_time_sum_ms=round(float(dur[red].sum()) / 1e3, 2),
      wait_sum_ms=round(float(wait.sum()) / 1e3, 2))))
# timeline: fraction of CTAs in expand / reduce over 10 time slices
edges = np.linspace(0, span, 11)
row = []
for i in range(10):
    a, b = edges[i] * 1e3, edges[i + 1] * 1e3
    ov = np.clip(np.minimum(tr[:, 3], b) - np.maximum(tr[:, 1], a), 0, None)
    row.append((round(float(ov[~red].sum() / (b - a)), 1), round(float(ov[red].sum() / (b - a)), 1)))
print("active CTAs (expand, reduce) per tenth:", row)
