#!/usr/bin/env python
"""bench.py -- the driver's benchmark contract (one JSON line on rank 0).

Workload (BASELINE.json configs[1]): LiveJournal-shaped R-MAT graph,
n = 4,847,571 vertices, m = 68,993,773 edges, valued (edge values U(0,1]), fp32.
Step: one tiled-composite SpMV y = A x through spmv_execute in the execution the performance model
picks (two-phase tiles on c2: one persistent launch; one-pass tiles: x relabel + every tile launch),
inputs resident in HBM.  Metric: SpMV GFLOP/s (= 2 m / step time); HBM GB/s and the PageRank /
HITS / RWR iteration rates on the same graph are reported beside it.
N > 1 (torchrun): every rank runs its own replica of the workload (independent problems, no
data-path collective): weak scaling, value = total flops of all ranks / max-over-ranks time.
At every N, key "c4_pagerank": BASELINE configs[3] (it-2004-shaped, 1.15 B edges) PageRank
row-partitioned over all ranks (strong scaling; one allgather of the next x per iteration), each
rank generating its own rows on its GPU; device time max over ranks, plus its end-to-end time.
`--impl reference` times the fp64 CPU oracle (the only reference this paper-only tier has).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SpMV GFLOP/s and HBM GB/s vs 8 TB/s; PageRank iters/s at 1/2/4/8 B200"
WORKLOAD = "c2: LiveJournal-shaped R-MAT s23 (a,b,c,d)=(.50,.20,.20,.10), n=4847571, m=68993773, valued fp32"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.samples, self.stop = index, [], threading.Event()
        self.marks = []

    def _nvml(self):
        """NVML (what nvidia-smi reads) polled every 5 ms: enough samples inside a sub-second timed
        region; the device is matched by PCI bus id (CUDA and NVML orderings may differ)."""
        try:
            import pynvml as N
            import torch
            N.nvmlInit()
            pr = torch.cuda.get_device_properties(self.index)
            bus = "%08x:%02x:%02x.0" % (pr.pci_domain_id, pr.pci_bus_id, pr.pci_device_id)
            h = N.nvmlDeviceGetHandleByPciBusId(bus)
            mx = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
            get_reasons = getattr(N, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                N.nvmlDeviceGetCurrentClocksThrottleReasons
        except Exception:
            return False
        bits = [0x8, 0x40, 0x20, 0x4]     # hw_slowdown, hw_thermal, sw_thermal, sw_power_cap
        while not self.stop.is_set():
            try:
                sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
                r = get_reasons(h)
                flags = ",".join("Active" if r & b else "Not Active" for b in bits)
                self.samples.append((time.time(), f"{sm}, {mx}, {flags}"))
            except Exception:
                pass
            time.sleep(0.005)
        return True

    def _run(self):
        if self._nvml():
            return
        while not self.stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                self.samples.append((time.time(), out))
            except Exception:
                pass
            time.sleep(0.05)

    def __enter__(self):
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.t.join(timeout=10)

    def summary(self, t0, t1):
        rows = [s for (t, s) in self.samples if t0 <= t <= t1] or [s for (_, s) in self.samples]
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            f = [x.strip() for x in r.split(",")]
            try:
                sm.append(float(f[0])); mx = max(mx, float(f[1]))
                for i, nm in enumerate(names):
                    if f[2 + i].lower().startswith("active"):
                        reasons.add(nm)
            except Exception:
                continue
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def measure_traffic(kernel):
    """DRAM bytes (read + write) of the last captured launch of `kernel`, or None."""
    import shutil
    ncu = shutil.which("ncu") or "/usr/local/cuda/bin/ncu"
    if not os.path.exists(ncu):
        return None
    try:
        out = subprocess.run([ncu, "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum", "-k",
                              f"regex:{kernel}", "-s", "2", "-c", "1", "--csv", sys.executable,
                              os.path.join(ROOT, "bench", "ncu_traffic.py")],
                             capture_output=True, text=True, timeout=300).stdout
        tot, unit = 0.0, {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        import csv as _csv
        for row in _csv.reader(l for l in out.splitlines() if l.startswith('"')):
            if len(row) > 3 and row[-3].startswith("dram__bytes_"):
                tot += float(row[-1].replace(",", "")) * unit.get(row[-2], 1)
        return tot or None
    except Exception:
        return None


def load_workload():
    import graphgen
    G = graphgen.make_graph("c2")
    val = graphgen.edge_values(G.keys, seed=graphgen.SEED_VAL, mode=1)
    x = graphgen.uniform_f32(G.n, seed=graphgen.SEED_X)
    return G, val, x


def reference_arm(args):
    """fp64 CPU oracle, as it stands, on this box's host cores."""
    import oracle
    G, val, x = load_workload()
    oracle.spmv(G.row_ptr, G.col, val, x)        # warm (page-in)
    for _ in range(max(0, min(args.warmup, 1))):
        oracle.spmv(G.row_ptr, G.col, val, x)
    steps = max(1, min(args.steps, 5))
    t0 = time.perf_counter()
    for _ in range(steps):
        oracle.spmv(G.row_ptr, G.col, val, x)
    dt = (time.perf_counter() - t0) / steps
    v = 2.0 * G.m / dt / 1e9
    cores = len(os.sched_getaffinity(0))
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 3), "unit": "GFLOP/s",
            "n_gpus": args.gpus, "steps": steps, "warmup": args.warmup, "ms_per_step": round(dt * 1e3, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": WORKLOAD},
            "cpu_baseline": {"value": round(v, 3), "unit": "GFLOP/s", "cores": cores, "kind": "oracle",
                             "sample": f"full c2 SpMV x {steps} (fp64 CSR, OpenMP over rows)"},
            "e2e": {"value": round(v, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def c4_pagerank_leg(args, pkg, local, rank, world):
    import torch
    import torch.distributed as dist
    import graphgen
    out = {}
    t_g = time.time()
    dg = graphgen.DeviceGraph("c4", device=local)
    n, m = dg.n, dg.m
    od, idg = dg.degrees()
    owner = pkg.bitonic_partition(idg.astype(np.int64), world)
    ids, rp, col = dg.owned_rows(graphgen.KIND_AT, owner, rank)
    del owner
    keys = dg.keys() if world == 1 else None
    dg.close()
    gen_s = time.time() - t_g

    def mx(v):
        if world == 1:
            return v
        tt = torch.tensor([v], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return float(tt.item())

    comm = pkg.Comm.from_torch(local) if world > 1 else pkg.Comm(0, 1, b"\0" * 128, local)
    t_b = time.time()
    s = pkg.Solver.local("pagerank", n, ids, rp, col, out_degree=od[ids], device=local, comm=comm)
    build_s = mx(time.time() - t_b)
    del rp, col
    s.run()                                   # warm-up
    info = s.run()
    ms = mx(info["ms_total"])
    # end to end through the API: the solve plus the result on the host (the one-time gather of
    # every rank's rows and its D2H copy), host wall clock, max over ranks
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ie = s.run()
    p = s.result()
    e2e_ms = mx((time.perf_counter() - t0) * 1e3)
    out["c4_pagerank"] = {
        "workload": f"c4: it-2004-shaped Graph500 R-MAT s26, n={n}, m={m}, pattern",
        "n_gpus": world, "scaling": "strong", "parallelism": f"row-partitioned x{world} (allgather)",
        "iterations": info["iterations"], "iters_per_s": round(1e3 * info["iterations"] / ms, 1),
        "ms_per_iter": round(ms / max(info["iterations"], 1), 3),
        "phase_us": [round(mx(v), 1) for v in info["phase_us"]],
        "predicted_us_per_iter_rank": round(info["predicted_us_per_iter"], 1),
        "e2e": {"value": round(1e3 * ie["iterations"] / e2e_ms, 1), "unit": "iters/s",
                "ms": round(e2e_ms, 2), "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 4 * n,
                "note": "solve + result gather to host; the graph is resident (built once, L98)"},
        "gen_s": round(mx(gen_s), 1), "build_s": round(build_s, 1),
        "sum_p": round(float(np.sum(p, dtype=np.float64)), 6)}
    s.close()
    comm.close()
    if world == 1:
        # the single-GPU solver (no exchange, its own tile plan) on the same graph
        G4 = graphgen.graph_from_keys("c4", n, keys)
        del keys
        t_b = time.time()
        s4 = pkg.Solver("pagerank", G4.n, G4.row_ptr, G4.col, device=local)
        b4 = time.time() - t_b
        s4.run()
        i4 = s4.run()
        out["c4_pagerank_iters_per_s"] = round(1e3 * i4["iterations"] / i4["ms_total"], 1)
        out["c4_pagerank_iterations"] = i4["iterations"]
        out["c4_pagerank_us_per_iter"] = round(i4["us_per_iter"], 1)
        out["c4_pagerank_predicted_us_per_iter"] = round(i4["predicted_us_per_iter"], 1)
        out["c4_workload"] = f"it-2004-shaped Graph500 R-MAT s26, n={G4.n}, m={G4.m}, pattern, 1 GPU"
        out["c4_gen_s"] = round(gen_s, 1)
        out["c4_build_s"] = round(b4, 1)
        s4.close()
        del G4
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-extras", action="store_true", help="skip PageRank/HITS/RWR and cpu_baseline")
    ap.add_argument("--no-c4", action="store_true", help="skip the c4 PageRank leg (about 5 minutes)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        if rank == 0:
            reference_arm(args)
        return

    import torch
    import torch.distributed as dist
    import graphgen
    import paper_1103_2405_b200 as pkg

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    G, val, x = load_workload()
    plan = pkg.Plan(G.n, G.n, G.row_ptr, G.col, val, device=local)
    st = plan.stats()
    xt = torch.from_numpy(x).cuda()
    yt = torch.empty(G.n, device="cuda")
    stream = torch.cuda.current_stream()

    plan.execute(xt, yt)
    torch.cuda.synchronize()

    for _ in range(args.warmup):
        plan.execute(xt, yt)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        # ~1 s soak so the clock sampler sees the kernel under load
        t_soak = time.time()
        while time.time() - t_soak < 1.0:
            for _ in range(50):
                plan.execute(xt, yt)
            torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.time()
        # the K timed steps in 5 batches with an event at each boundary (median and
        # mean of 5 batches are reported beside the whole-run value; events do not sync)
        nb = 5 if args.steps >= 5 else 1
        bounds = [args.steps * i // nb for i in range(nb + 1)]
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(nb - 1)]
        e0.record(stream)
        for i in range(nb):
            for _ in range(bounds[i + 1] - bounds[i]):
                plan.execute(xt, yt)
            if i < nb - 1:
                ev[i].record(stream)
        e1.record(stream)
        torch.cuda.synchronize()
        t1 = time.time()
        if world > 1:
            dist.barrier()
    ms = e0.elapsed_time(e1) / args.steps
    marks = [e0] + ev + [e1]
    batch_ms = [marks[i].elapsed_time(marks[i + 1]) / max(bounds[i + 1] - bounds[i], 1) for i in range(nb)]
    if world > 1:
        tt = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    value = world * 2.0 * G.m / (ms * 1e-3) / 1e9
    alg_bytes = 8 * G.m + 12 * G.n
    hbm_gbs = alg_bytes / (ms * 1e-3) / 1e9

    # per-launch device times (CUDA events between launches on the same stream)
    nl = plan.launches
    per = np.zeros(nl, np.float64)
    buf = (np.zeros(nl, np.float32))
    reps = max(10, args.steps // 10)
    import ctypes
    for _ in range(reps):
        pkg._capi.check(pkg.lib().spmv_execute_timed(plan._h, ctypes.c_void_p(xt.data_ptr()),
                                                      ctypes.c_void_p(yt.data_ptr()),
                                                      ctypes.c_void_p(stream.cuda_stream),
                                                      buf.ctypes.data, nl), "spmv_execute_timed")
        per += buf
    per /= reps
    if st["two_phase"]:
        # two-phase tiles: one persistent launch, no x relabel; its algorithmic
        # bytes are the whole product's (8 m + 12 n valued)
        launch_bytes = [8.0 * G.m + 12.0 * G.n]
        launch_names = ["pb_spmv(two-phase tiles)"]
        launch_nnz = [G.m]
    else:
        # launch 0 = x permutation (12 B per column), then the non-empty tiles in order
        tiles = [t for t in range(st["num_tiles"] + 1) if st["tile_nnz"][t] > 0 or t == st["num_tiles"]]
        launch_bytes = [12.0 * G.n]
        launch_names = ["permute_x"]
        launch_nnz = [0]
        for t in tiles[: nl - 1]:
            launch_nnz.append(st["tile_nnz"][t])
            width = st["tile_col_hi"][t] - st["tile_col_lo"][t]
            launch_bytes.append(8.0 * st["tile_nnz"][t] + 8.0 * st["tile_rows"][t] + 4.0 * width)
            launch_names.append(f"tc_spmv_tile[{t}]" + ("(smem x)" if st["tile_staged"][t] else "(L1/L2 x)"))
    dom = int(np.argmax(per))
    peak, peak_src = peaks()
    ach = launch_bytes[dom] / (per[dom] * 1e-3) / 1e9
    roofline = {"bound": "hbm", "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
                "frac": round(ach / peak, 4), "traffic": None, "kernel": launch_names[dom],
                "kernel_share": round(float(per[dom] / per.sum()), 3), "peak_source": peak_src,
                "per_launch_us": [round(float(v) * 1e3, 2) for v in per],
                "launch_names": launch_names}
    # the ceiling that binds on B200: random x gathers per second, measured by
    # bench/probe/probe.cu on an x of the closest size (skewed columns, L1-allocating loads)
    try:
        best = None
        with open(os.path.join(ROOT, "profiles", "r01_probe_gather.jsonl")) as f:
            for ln in f:
                r = json.loads(ln)
                if r.get("probe") == "gather" and r.get("dist") == "skew" and r.get("mode") == 0:
                    if best is None or abs(np.log(r["S"] / G.n)) < abs(np.log(best["S"] / G.n)):
                        best = r
        if best is not None and launch_nnz[dom] > 0 and not st["two_phase"]:
            g_ach = launch_nnz[dom] / (per[dom] * 1e-3) / 1e9
            roofline["gather"] = {"achieved_G_per_s": round(g_ach, 1), "probe_G_per_s": best["Ggather_s"],
                                  "frac": round(g_ach / best["Ggather_s"], 3),
                                  "probe": "profiles/r01_probe_gather.jsonl skew S=%d" % best["S"]}
    except Exception:
        pass
    # DRAM traffic of the dominant kernel, measured in this run: one ncu pass (dram bytes only)
    # over a fresh process that builds the same plan and launches it three times
    if rank == 0 and world == 1 and not os.environ.get("TCSPMV_BENCH_NO_NCU"):
        tr = measure_traffic("pb_spmv" if st["two_phase"] else "tc_spmv_tile")
        if tr:
            roofline["traffic"] = tr
            roofline["traffic_source"] = "ncu dram__bytes_read.sum + dram__bytes_write.sum, this run (bench/ncu_traffic.py)"
            # effective DRAM bytes per stored entry vs the minimum 8 + 12 n / m
            roofline["dram_bytes_per_nnz"] = round(tr / G.m, 2)
            roofline["min_bytes_per_nnz"] = round(8 + 12 * G.n / G.m, 2)

    # end to end through the public API with host buffers: spmv_execute_host_batch copies every
    # step's x in (pinned H2D) and its y out (D2H) inside the timed region, overlapping the copies
    # of neighbouring steps with the product (two copy streams, double-buffered)
    e2e_steps = min(max(5, args.steps // 10), 32)
    xh = torch.from_numpy(x).unsqueeze(0).expand(e2e_steps, G.n).contiguous().pin_memory()
    yh = torch.empty((e2e_steps, G.n), dtype=torch.float32).pin_memory()

    def e2e_call(cnt):
        pkg._capi.check(pkg.lib().spmv_execute_host_batch(plan._h, ctypes.c_void_p(xh.data_ptr()),
                                                           ctypes.c_void_p(yh.data_ptr()), cnt,
                                                           ctypes.c_void_p(stream.cuda_stream)), "e2e")
    e2e_call(e2e_steps)        # warm-up over every pinned page (first DMA to a page maps it)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    e2e_call(e2e_steps)
    f1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = f0.elapsed_time(f1) / e2e_steps
    if world > 1:
        tt = torch.tensor([e2e_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = float(tt.item())
    e2e = {"value": round(world * 2.0 * G.m / (e2e_ms * 1e-3) / 1e9, 3), "unit": "GFLOP/s",
           "h2d_bytes_per_step": 4 * G.n, "d2h_bytes_per_step": 4 * G.n,
           "ms_per_step": round(e2e_ms, 4)}

    extras, cpu = {}, None
    if rank == 0 and world == 1 and not args.no_extras:
        # the other execution of the same format on the same workload: the one-pass tiles (x relabel
        # + tile launches); the model picks between the two by predicted time (DESIGN 7c)
        po = pkg.Plan(G.n, G.n, G.row_ptr, G.col, val, device=local, two_phase=0)
        for _ in range(10):
            po.execute(xt, yt, stream=stream)
        h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        h0.record(stream)
        for _ in range(200):
            po.execute(xt, yt, stream=stream)
        h1.record(stream)
        torch.cuda.synchronize()
        per_o = np.zeros(po.launches, np.float64)
        bo = np.zeros(po.launches, np.float32)
        for _ in range(20):
            pkg._capi.check(pkg.lib().spmv_execute_timed(po._h, ctypes.c_void_p(xt.data_ptr()),
                                                          ctypes.c_void_p(yt.data_ptr()),
                                                          ctypes.c_void_p(stream.cuda_stream), bo.ctypes.data,
                                                          po.launches), "spmv_execute_timed")
            per_o += bo
        per_o /= 20
        tile_us = float(per_o[1:].sum()) * 1e3
        sto = po.stats()
        extras["one_pass"] = {"us_per_step": round(h0.elapsed_time(h1) * 1e3 / 200, 2),
                              "launch_us": [round(float(v) * 1e3, 2) for v in per_o],
                              "tile_frac_of_peak": round((8 * G.m + 12 * G.n) / (tile_us * 1e-6) / 1e9 / roofline["peak"], 4),
                              "predicted_us": round(sto["predicted_us"], 1), "wl": sto["wl"], "num_tiles": sto["num_tiles"]}
        po.close()
        # BASELINE configs[0] (R-MAT s16, ~1 M entries; L2-resident: launch/latency-bound, so
        # reported in microseconds, not against the roofline): SpMV and PageRank to 1e-6
        import graphgen
        G1 = graphgen.make_graph("c1")
        v1 = graphgen.edge_values(G1.keys, seed=graphgen.SEED_VAL, mode=1)
        p1 = pkg.Plan(G1.n, G1.n, G1.row_ptr, G1.col, v1, device=local)
        x1 = torch.from_numpy(graphgen.uniform_f32(G1.n, seed=graphgen.SEED_X)).cuda()
        y1 = torch.empty(G1.n, device="cuda")
        for _ in range(10):
            p1.execute(x1, y1, stream=stream)
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for _ in range(200):
            p1.execute(x1, y1, stream=stream)
        g1.record(stream)
        torch.cuda.synchronize()
        extras["c1_spmv_us"] = round(g0.elapsed_time(g1) * 1e3 / 200, 2)
        extras["c1_spmv_gflops"] = round(2 * G1.m / (extras["c1_spmv_us"] * 1e3), 1)
        p1.close()
        s1 = pkg.Solver("pagerank", G1.n, G1.row_ptr, G1.col, device=local)
        s1.run()
        i1 = s1.run()
        extras["c1_pagerank_iterations"] = i1["iterations"]
        extras["c1_pagerank_us_per_iter"] = round(i1["us_per_iter"], 2)
        extras["c1_pagerank_iters_per_s"] = round(1e6 / i1["us_per_iter"], 1)
        s1.close()
        for algo in ("pagerank", "hits", "rwr"):
            s = pkg.Solver(algo, G.n, G.row_ptr, G.col, device=local)
            q = int(np.nonzero(np.diff(G.row_ptr) > 0)[0][0]) if algo == "rwr" else 0
            s.run(q)
            info = s.run(q)
            extras[f"{algo}_iters_per_s"] = round(1e3 * info["iterations"] / info["ms_total"], 1)
            extras[f"{algo}_iterations"] = info["iterations"]
            extras[f"{algo}_us_per_iter"] = round(info["us_per_iter"], 2)
            extras[f"{algo}_predicted_us_per_iter"] = round(info["predicted_us_per_iter"], 1)
            if algo == "rwr":
                # the paper's 25 random queries (L448), batched as one SpMM per iteration (f1)
                deg = np.diff(G.row_ptr) + np.bincount(G.col, minlength=G.n)
                rng = np.random.default_rng(graphgen.SEED_QUERY)
                qs = rng.choice(np.nonzero(deg > 0)[0], size=25, replace=False)
                s.run_batch(qs)
                bi = s.run_batch(qs)
                extras["rwr_batch25_us_per_iter"] = round(bi["us_per_iter"], 1)
                extras["rwr_batch25_query_iters_per_s"] = round(25 * 1e6 / bi["us_per_iter"], 1)
                # capacity: the SpMM's lanes are 32 queries wide, so a full batch costs the same pass
                q32 = rng.choice(np.nonzero(deg > 0)[0], size=32, replace=False)
                s.run_batch(q32)
                b32 = s.run_batch(q32)
                extras["rwr_batch32_us_per_iter"] = round(b32["us_per_iter"], 1)
                extras["rwr_batch32_query_iters_per_s"] = round(32 * 1e6 / b32["us_per_iter"], 1)
            s.close()
        # cpu_baseline: the oracle as it stands on this box's host cores, bounded sample
        import oracle
        oracle.spmv(G.row_ptr, G.col, val, x)
        reps_cpu, tc0 = 0, time.perf_counter()
        while time.perf_counter() - tc0 < 10.0:
            oracle.spmv(G.row_ptr, G.col, val, x)
            reps_cpu += 1
        dtc = (time.perf_counter() - tc0) / reps_cpu
        cpu = {"value": round(2.0 * G.m / dtc / 1e9, 3), "unit": "GFLOP/s",
               "cores": len(os.sched_getaffinity(0)), "kind": "oracle",
               "sample": f"full c2 SpMV repeated {reps_cpu}x over ~10 s (fp64 CSR, OpenMP over rows)"}
        # the paper-comparable one-thread CPU CSR run (SURVEY.md 8(d) "Oracle timing" (2))
        try:
            gomp = ctypes.CDLL("libgomp.so.1")
            gomp.omp_set_num_threads(1)
            reps1, tc0 = 0, time.perf_counter()
            while time.perf_counter() - tc0 < 5.0:
                oracle.spmv(G.row_ptr, G.col, val, x)
                reps1 += 1
            cpu["one_thread"] = {"value": round(2.0 * G.m * reps1 / (time.perf_counter() - tc0) / 1e9, 3),
                                 "unit": "GFLOP/s", "cores": 1,
                                 "sample": f"full c2 SpMV repeated {reps1}x over ~5 s, one OpenMP thread"}
        finally:
            gomp.omp_set_num_threads(len(os.sched_getaffinity(0)))

    # BASELINE configs[3]: PageRank on the it-2004-shaped graph (41.3 M vertices, 1.15 B edges, x
    # beyond L2), row-partitioned over all N ranks (Sec. 3.2; strong scaling: one graph):
    # every rank draws the graph on its own GPU (device generator, bit-identical to graphgen.c),
    # keeps its rows of A^T under the library's bitonic partition and builds its local solver
    # (spmv_solver_create_local); one allgather of the next x per iteration.  At N = 1 the same
    # path runs with a world-1 communicator, and the single-GPU solver (no exchange) beside it.
    if not args.no_extras and not args.no_c4:
        try:
            extras.update(c4_pagerank_leg(args, pkg, local, rank, world))
        except Exception as ex:
            extras["c4_error"] = str(ex)[:300]

    # row-partitioned PageRank over all ranks (Sec. 3.2): one NCCL allgather per iteration
    if world > 1 and not os.environ.get("TCSPMV_BENCH_NO_DIST"):
        try:
            comm = pkg.Comm.from_torch(local)
            sd = pkg.Solver("pagerank", G.n, G.row_ptr, G.col, device=local, comm=comm)
            sd.run()
            info = sd.run()
            tt = torch.tensor([info["ms_total"]], device="cuda", dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            extras["pagerank_dist_iters_per_s"] = round(1e3 * info["iterations"] / float(tt.item()), 1)
            extras["pagerank_dist_iterations"] = info["iterations"]
            extras["pagerank_dist_scaling"] = "strong (one graph over all ranks)"
            sd.close()
            # the needed-columns exchange on the same graph
            sn = pkg.Solver("pagerank", G.n, G.row_ptr, G.col, device=local, comm=comm, iter_kw=dict(exchange=1))
            sn.run()
            info = sn.run()
            tt = torch.tensor([info["ms_total"]], device="cuda", dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            extras["pagerank_dist_needed_iters_per_s"] = round(1e3 * info["iterations"] / float(tt.item()), 1)
            sn.close()
            comm.close()
        except Exception as ex:          # reported, never fatal for the replica measurement
            extras["pagerank_dist_error"] = str(ex)[:300]

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "GFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 5),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": WORKLOAD, "parallelism": f"replicas{world}",
                       "l2": "inputs larger than L2 (0.57 GB of col/val streamed per step); x (19 MB) L2-resident",
                       "plan": {k: st[k] for k in ("two_phase", "num_tiles", "tile_width", "wl", "tile_staged",
                                                     "n_workloads", "n_slots", "pb_groups", "pb_chunks",
                                                     "pb_bins", "one_pass_predicted_us",
                                                     "two_phase_predicted_us")}},
            "hbm_GBps_algorithmic": round(hbm_gbs, 1),
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(args.steps * nl),
            "clocks": clk.summary(t_soak, t1),
            "predicted_us": round(st["predicted_us"], 2),
            "plan_build_ms": round(st["build_ms"], 1),      # one-time, amortised, not in the step
            "batches_ms_per_step": {"n": nb, "median": round(float(np.median(batch_ms)), 5),
                                    "mean": round(float(np.mean(batch_ms)), 5)},
        }
        line.update(extras)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
