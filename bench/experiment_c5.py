#!/usr/bin/env python
"""c5 (BASELINE.json configs[4]): HITS on the uk-union-shaped graph -- Graph500 R-MAT
scale 28, n = 133,633,040, m = 5,507,679,822; the HITS block [[0, A^T], [A, 0]] has 267 M rows and
11.0 B entries (Eq. 8; multi-GPU web graphs, L202).

Route (nothing of size m ever exists whole on the host):
  1. the device generator draws the keys (graphgen.DeviceGraph, bit-identical to graphgen.c);
  2. the library's bitonic partition of the block rows by length (Sec. 3.2) into P slices;
  3. each slice's rows of the block come off the device (DeviceGraph.owned_rows) -> host CSR;
  4. P ranks on this one GPU each build their row-partitioned HITS solver from their slice
     (spmv_solver_create_local), one build at a time; by default they are slices of one solver
     sharing one exchange buffer (spmv_comm_create_slices: the exchange is ordering only), or
     (--transport loopback) each has its own buffer and pulls its peers' slots by device copies;
  5. K-1 and then K iterations at fixed k (spmv_solver_set_stop), device time max over ranks;
  6. parity: the oracle's fp64 product of the block with the GPU's iterate k-1, halves normalised
     (the paper's sum-1 rule, L440), against the GPU's iterate k -- every row.
With the loopback transport the P ranks' exchanges (device copies) and normalisation passes over
their whole buffers run P times on the one device: the per-phase split says how much of an
iteration that is; the slices transport does neither.

python bench/experiment_c5.py [--config c5] [--P 8] [--iters 12] [--out file.jsonl]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(config="c5", P=8, iters=12, parity=True, transport="slices"):
    """The whole route; returns the record (parity under rec["parity"] when parity=True).
    transport "slices": the P ranks share one exchange buffer (spmv_comm_create_slices, no copies);
    "loopback": each rank has its own buffer and pulls its peers' slots (the multi-GPU protocol)."""
    args = argparse.Namespace(config=config, P=P, iters=iters, no_parity=not parity)
    import graphgen
    import paper_1103_2405_b200 as pkg

    rec = dict(config=args.config, P=args.P, iters=args.iters, transport=transport)
    t = time.time()
    dg = graphgen.DeviceGraph(args.config, device=0)
    rec["gen_s"] = round(time.time() - t, 1)
    n, m = dg.n, dg.m
    rec.update(n=n, m=m, block_rows=2 * n, block_entries=2 * m)
    print(f"[c5] generated n={n} m={m} in {rec['gen_s']} s", flush=True)
    t = time.time()
    lens = dg.row_lengths(graphgen.KIND_HITS)
    owner = pkg.bitonic_partition(lens, args.P)
    rec["partition_s"] = round(time.time() - t, 1)
    t = time.time()
    parts = [dg.owned_rows(graphgen.KIND_HITS, owner, q) for q in range(args.P)]
    rec["slices_s"] = round(time.time() - t, 1)
    rec["slice_entries"] = [int(p[1][-1]) for p in parts]
    rec["slice_rows"] = [int(len(p[0])) for p in parts]
    dg.close()
    del owner, lens
    print(f"[c5] partitioned + sliced in {rec['partition_s']} + {rec['slices_s']} s", flush=True)

    comms = pkg.Comm.slices(args.P, 0) if transport == "slices" else pkg.Comm.loopback(args.P, 0)
    out = [None] * args.P
    err = []
    build_s = [0.0] * args.P
    K = args.iters
    gate = threading.Barrier(args.P)

    def body(r):
        try:
            ids, rp, col = parts[r]
            t0 = time.time()
            s = pkg.Solver.local("hits", n, ids, rp, col, device=0, comm=comms[r],
                                 iter_kw=dict(hits_norm=1, fixed_iters=max(K - 1, 1)))
            build_s[r] = time.time() - t0
            parts[r] = None if args.no_parity else parts[r]
            gate.wait()
            st = s.stats()
            s.run(0, stream=0)                          # warm-up (graph of kernels, first touch)
            res = {}
            if K > 1:
                i1 = s.run(0, stream=0)
                v1 = s.result()
                res["prev"] = (i1, v1 if r == 0 else None)
            s.set_stop(fixed_iters=K)
            i2 = s.run(0, stream=0)
            v2 = s.result()
            res["last"] = (i2, v2 if r == 0 else None)
            res["stats"] = {k: st[k] for k in ("n_rows", "nnz", "num_tiles", "n_slots", "predicted_us", "build_ms",
                                               "device_bytes")}
            s.close()
            out[r] = res
        except BaseException as ex:   # noqa: BLE001
            err.append(ex)
            try:
                gate.abort()
            except Exception:
                pass

    th = [threading.Thread(target=body, args=(r,)) for r in range(args.P)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    for c in comms:
        c.close()
    if err:
        raise err[0]
    # the loopback builds run one at a time: the last rank's create call spans all of them
    rec["build_s_all_ranks"] = round(max(build_s), 1)
    rec["build_ms_per_rank_plan"] = None
    i2 = [o["last"][0] for o in out]
    ms = max(i["ms_total"] for i in i2)
    rec["iterations"] = i2[0]["iterations"]
    rec["ms_total_max_over_ranks"] = round(ms, 3)
    rec["ms_per_iter"] = round(ms / max(i2[0]["iterations"], 1), 3)
    rec["iters_per_s"] = round(1e3 * i2[0]["iterations"] / ms, 2)
    rec["phase_us_rank0"] = [round(v, 1) for v in i2[0]["phase_us"]]
    rec["phase_us_max"] = [round(max(i["phase_us"][k] for i in i2), 1) for k in range(3)]
    rec["predicted_us_per_iter_rank_max"] = round(max(i["predicted_us_per_iter"] for i in i2), 1)
    rec["plan"] = [o["stats"] for o in out]
    rec["build_ms_per_rank_plan"] = [round(o["stats"]["build_ms"], 1) for o in out]
    # algorithmic bytes per iteration (HITS block, pattern): 4 B per entry + 12 B per row,
    # plus 20 B per row for the epilogue / normalisation
    alg = 4 * 2 * m + 12 * 2 * n + 20 * 2 * n
    rec["hbm_GBps_algorithmic"] = round(alg / (ms / max(i2[0]["iterations"], 1) * 1e-3) / 1e9, 1)
    print(f"[c5] {rec['iterations']} iterations, {rec['ms_per_iter']} ms each", flush=True)

    if not args.no_parity and K > 1:
        import oracle
        a1, h1 = out[0]["prev"][1]
        a2, h2 = out[0]["last"][1]
        x = np.concatenate([a1, h1]).astype(np.float32)
        y = np.zeros(2 * n, np.float64)
        b = np.zeros(2 * n, np.float64)
        t = time.time()
        for ids, rp, col in parts:
            yq, bq = oracle.spmv(rp, col, None, x)
            y[ids] = yq
            b[ids] = bq
        rec["oracle_spmv_s"] = round(time.time() - t, 1)
        ra = y[:n] / y[:n].sum()
        rh = y[n:] / y[n:].sum()
        da = np.abs(a2.astype(np.float64) - ra)
        dh = np.abs(h2.astype(np.float64) - rh)
        rec["parity"] = dict(
            rule="one HITS step from the GPU's iterate k-1: oracle fp64 block product, sum-1 halves (L440), every row",
            l1_a=float(da.sum()), l1_h=float(dh.sum()),
            max_rel_a=float((da / np.maximum(ra, 1e-300))[ra > 0].max()) if (ra > 0).any() else 0.0,
            max_rel_h=float((dh / np.maximum(rh, 1e-300))[rh > 0].max()) if (rh > 0).any() else 0.0,
            zero_rows_exact=bool(np.all(a2[ra == 0] == 0) and np.all(h2[rh == 0] == 0)),
            ok=bool(da.sum() < 1e-6 and dh.sum() < 1e-6))
        print(f"[c5] parity {rec['parity']}", flush=True)
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--P", type=int, default=8)
    ap.add_argument("--iters", type=int, default=12)
    ap.add_argument("--out", default=None)
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--transport", default="slices", choices=["slices", "loopback"])
    args = ap.parse_args()
    rec = run(args.config, args.P, args.iters, not args.no_parity, args.transport)
    line = json.dumps(rec)
    print(line, flush=True)
    if args.out:
        with open(args.out, "a") as f:
            f.write(line + "\n")


if __name__ == "__main__":
    main()
