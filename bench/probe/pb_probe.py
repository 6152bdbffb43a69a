"""Feasibility probe (not the product, not a bench line): gather-free two-phase SpMV (pb_probe.cu).

Builds the phase-1 chunk/run tables and the phase-2 bin/slab tables with numpy, checks the tables
with a numpy emulation on the CPU (--emulate), and on the GPU times one SpMV (all groups) and
compares y with a float64 CSR product.
Usage: python bench/probe/pb_probe.py c2 [G] [--pattern] [--emulate]"""
import ctypes
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import graphgen  # noqa: E402

CHUNK_DT = np.dtype([("e0", "<i8"), ("n", "<i4"), ("col0", "<i4"), ("run0", "<i4"), ("nrun", "<i4")])
RUN_DT = np.dtype([("start", "<i4"), ("len", "<i4"), ("goff", "<i8")])
BIN_DT = np.dtype([("roff", "<i8"), ("rlen", "<i4"), ("row0", "<i4"), ("nrows", "<i4"), ("slab0", "<i4"),
                   ("nslab", "<i4"), ("nheavy", "<i4"), ("hoff", "<i8"), ("plen", "<i4"), ("pad2", "<i4")])
SLAB_DT = np.dtype([("poff", "<i8"), ("w", "<i4"), ("mode", "<i4")])


def build(rp, col, n, G=4, C=8192, RB=24576, RROWS=8192, WMAX=64):
    t0 = time.time()
    m = len(col)
    rowlen = np.diff(rp)
    rperm = np.argsort(-rowlen, kind="stable")
    rank = np.empty(n, np.int64)
    rank[rperm] = np.arange(n)
    rnew = rank[np.repeat(np.arange(n, dtype=np.int64), rowlen)]     # new row of every entry (CSR order)
    nlen = rowlen[rperm]
    cum = np.concatenate([[0], np.cumsum(nlen)])
    # row bins: <= RB partials and <= RROWS rows
    b0 = []
    r = 0
    while r < n:
        end = int(np.searchsorted(cum, cum[r] + RB, "right")) - 1
        end = min(max(end, r + 1), r + RROWS, n)
        b0.append(r)
        r = end
    b0 = np.array(b0 + [n], np.int64)
    nb = len(b0) - 1
    bin_rows = np.diff(b0)
    group_of_bin = np.minimum(G - 1, cum[b0[:-1]] * G // max(m, 1))
    group_of_bin = np.maximum.accumulate(group_of_bin)
    bin_of_row = np.repeat(np.arange(nb, dtype=np.int64), bin_rows)
    e_bin = bin_of_row[rnew]
    e_grp = group_of_bin[e_bin]
    # phase 1 order: (group, col, row)
    key = (e_grp << 50) | (col.astype(np.int64) << 25) | rnew
    o1 = np.argsort(key, kind="stable")
    del key
    g1 = e_grp[o1]
    c1 = col[o1].astype(np.int64)
    b1 = e_bin[o1]
    ge = np.searchsorted(g1, np.arange(G + 1))
    # chunks: <= C entries, column span < 65536, inside one group
    cs = []
    for g in range(G):
        s, e = int(ge[g]), int(ge[g + 1])
        while s < e:
            end = min(s + C, e, int(np.searchsorted(c1[s:e], c1[s] + 65536)) + s)
            cs.append(s)
            s = end
    cs = np.array(cs + [m], np.int64)
    nch = len(cs) - 1
    ch_of = np.repeat(np.arange(nch, dtype=np.int64), np.diff(cs))
    # stage position: inside the chunk by (bin, csc order)
    o2 = np.argsort(ch_of * nb + b1, kind="stable")
    dest = np.empty(m, np.int64)
    dest[o2] = np.arange(m) - cs[ch_of[o2]]
    # global buffer position: (bin, chunk, csc order)
    o3 = np.argsort(b1 * nch + ch_of, kind="stable")
    gpos = np.empty(m, np.int64)
    gpos[o3] = np.arange(m)
    # runs = maximal (chunk, bin) groups in o2 order
    kk = (ch_of * nb + b1)[o2]
    rstart = np.concatenate([[0], np.nonzero(np.diff(kk))[0] + 1]) if m else np.zeros(0, np.int64)
    rlen = np.diff(np.concatenate([rstart, [m]]))
    first = o2[rstart]                      # o1-positions of each run's first entry
    runs = np.zeros(len(rstart), RUN_DT)
    runs["start"] = dest[first]
    runs["len"] = rlen
    # regions start 16-byte aligned: padded buffer position of every entry
    bs0 = np.searchsorted(b1[o3], np.arange(nb + 1))
    rl = np.diff(bs0)
    rs_pad = np.concatenate([[0], np.cumsum((rl + 3) // 4 * 4)])
    gbase = rs_pad[np.searchsorted(group_of_bin, np.arange(G + 1))]        # group buffer bases
    gpos = gpos - bs0[b1] + rs_pad[b1]
    runs["goff"] = gpos[first] - gbase[g1[first]]
    run_ch = ch_of[first]
    # run index (within its chunk) of every stage position, chunk-major (PB_FLAT == 2)
    run_of_t = np.searchsorted(rstart, np.arange(m), "right") - 1
    rid = (run_of_t - np.searchsorted(run_ch, ch_of[o2], "left")).astype(np.uint16)
    chunks = np.zeros(nch, CHUNK_DT)
    chunks["e0"] = cs[:-1]
    chunks["n"] = np.diff(cs)
    chunks["col0"] = c1[cs[:-1]] if nch else 0
    chunks["run0"] = np.searchsorted(run_ch, np.arange(nch))
    chunks["nrun"] = np.searchsorted(run_ch, np.arange(nch), "right") - chunks["run0"]
    colrel = c1 - c1[cs[ch_of]]
    assert colrel.max(initial=0) < 65536 and dest.max(initial=0) < 65536
    cd = (colrel | (dest << 16)).astype(np.uint32)
    gc = np.searchsorted(g1[cs[:-1]], np.arange(G + 1)).astype(np.int32)
    # bins / regions
    bins = np.zeros(nb, BIN_DT)
    bins["roff"] = rs_pad[:-1] - gbase[group_of_bin]
    bins["rlen"] = rl
    assert bins["rlen"].max(initial=0) < 65535
    bins["row0"] = b0[:-1]
    bins["nrows"] = bin_rows
    heavy = nlen > WMAX
    nh = np.zeros(nb, np.int64)
    np.add.at(nh, bin_of_row[heavy], 1)
    bins["nheavy"] = nh
    nl = bin_rows - nh
    nsl = (nl + 31) // 32
    bins["nslab"] = nsl
    bins["slab0"] = np.concatenate([[0], np.cumsum(nsl)[:-1]])
    gb = np.searchsorted(group_of_bin, np.arange(G + 1)).astype(np.int32)
    # pos layout: per bin, its heavy rows row-major (offset cum[r] - cum[row0]) then its light slabs
    hlen = cum[b0[:-1] + nh] - cum[b0[:-1]]
    S = int(nsl.sum())
    slab_bin = np.repeat(np.arange(nb, dtype=np.int64), nsl)
    slab_row0 = (b0[:-1] + nh)[slab_bin] + 32 * (np.arange(S) - bins["slab0"][slab_bin])
    w = nlen[slab_row0] if S else np.zeros(0, np.int64)
    slabs = np.zeros(S, SLAB_DT)
    slabs["w"] = w
    blk = hlen + np.bincount(slab_bin, weights=32 * w, minlength=nb).astype(np.int64)   # pos per bin
    blk = (blk + 7) // 8 * 8                                         # 16-byte aligned blocks
    bstart = np.concatenate([[0], np.cumsum(blk)[:-1]])
    bins["hoff"] = bstart
    bins["plen"] = blk
    within = np.concatenate([[0], np.cumsum(32 * w)[:-1]]) - np.concatenate([[0], np.cumsum(32 * w)])[bins["slab0"][slab_bin]]
    slabs["poff"] = (bstart + hlen)[slab_bin] + within
    npos = int(blk.sum())
    # positions: row's partials ordered by region position
    lp = gpos - rs_pad[b1]                                          # o1 order
    rr = rnew[o1]
    o4 = np.lexsort((lp, rr))
    rr4, lp4 = rr[o4], lp[o4]
    k = np.arange(m) - cum[rr4]
    bi = bin_of_row[rr4]
    is_h = heavy[rr4]
    lr = rr4 - b0[bi] - nh[bi]                                      # light row index in the bin
    slab = bins["slab0"][bi] + np.maximum(lr, 0) // 32
    lane = np.maximum(lr, 0) % 32
    idx = np.where(is_h, bstart[bi] + cum[rr4] - cum[b0[bi]] + k,
                   slabs["poff"][np.minimum(slab, max(S - 1, 0))] + k * 32 + lane)
    pos = np.empty(npos, np.uint16)
    pad_bin = np.repeat(np.arange(nb), blk)
    pos[:] = bins["rlen"][pad_bin].astype(np.uint16)                # padding -> region sentinel (zero)
    pos[idx] = lp4.astype(np.uint16)
    perm_val = o1                                                   # val in phase-1 order = val[o1]
    info = dict(m=m, n=n, G=G, chunks=nch, runs=len(runs), bins=nb, slabs=S, npos=npos,
                mean_run=round(m / max(len(runs), 1), 1), max_group_entries=int(np.diff(gbase).max()),
                build_s=round(time.time() - t0, 1))
    return dict(rid=rid, cd=cd, perm_val=perm_val, nlen=nlen.astype(np.int32), rcum=cum.astype(np.int64), chunks=chunks, runs=runs, gc=gc, gb=gb, bins=bins, slabs=slabs,
                pos=pos, rperm=rperm, ge=ge, info=info)


def emulate(T, x, val_o1):
    """numpy execution of the two phases (table check)."""
    n = T["info"]["n"]
    buf = np.zeros(T["info"]["max_group_entries"] + 1, np.float64)
    y = np.zeros(n, np.float64)
    for g in range(T["info"]["G"]):
        for ci in range(T["gc"][g], T["gc"][g + 1]):
            c = T["chunks"][ci]
            cdv = T["cd"][c["e0"]:c["e0"] + c["n"]].astype(np.int64)
            v = x[c["col0"] + (cdv & 0xFFFF)].astype(np.float64)
            if val_o1 is not None:
                v = v * val_o1[c["e0"]:c["e0"] + c["n"]]
            st = np.zeros(c["n"])
            st[cdv >> 16] = v
            for ru in T["runs"][c["run0"]:c["run0"] + c["nrun"]]:
                buf[ru["goff"]:ru["goff"] + ru["len"]] = st[ru["start"]:ru["start"] + ru["len"]]
        for bi in range(T["gb"][g], T["gb"][g + 1]):
            b = T["bins"][bi]
            reg = np.concatenate([buf[b["roff"]:b["roff"] + b["rlen"]], [0.0]])
            for r in range(b["nheavy"]):
                o = b["hoff"] + T["rcum"][b["row0"] + r] - T["rcum"][b["row0"]]
                ln = T["nlen"][b["row0"] + r]
                y[b["row0"] + r] = reg[T["pos"][o:o + ln].astype(np.int64)].sum()
            for s in range(b["nslab"]):
                sl = T["slabs"][b["slab0"] + s]
                P = T["pos"][sl["poff"]:sl["poff"] + 32 * sl["w"]].astype(np.int64)
                acc = reg[P.reshape(sl["w"], 32).T].sum(axis=1)
                for lane in range(32):
                    r = b["nheavy"] + s * 32 + lane
                    if r < b["nrows"]:
                        y[b["row0"] + r] = acc[lane]
    return y


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
    G = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 4
    pattern = "--pattern" in sys.argv
    Gr = graphgen.make_graph(cfg)
    rp, col = Gr.row_ptr, Gr.col
    val = None if pattern else graphgen.edge_values(Gr.keys)
    x = graphgen.uniform_f32(Gr.n, seed=3)
    T = build(rp, col, Gr.n, G=G, C=int(os.environ.get("PB_C", 8192)), RB=int(os.environ.get("PB_RB", 24576)))
    print(json.dumps(T["info"]), file=sys.stderr, flush=True)
    val_o1 = None if pattern else np.ascontiguousarray(val[T["perm_val"]])
    # reference (fp64 CSR), in the new row order
    rows = np.repeat(np.arange(Gr.n), np.diff(rp))
    yref = np.zeros(Gr.n)
    np.add.at(yref, rows, (val.astype(np.float64) if val is not None else 1.0) * x[col].astype(np.float64))
    babs = np.zeros(Gr.n)
    np.add.at(babs, rows, np.abs((val.astype(np.float64) if val is not None else 1.0) * x[col].astype(np.float64)))
    yref, babs = yref[T["rperm"]], babs[T["rperm"]]
    if "--emulate" in sys.argv:
        y = emulate(T, x, val_o1)
        print(json.dumps(dict(cfg=cfg, emulate=True, ok=bool(np.all(np.abs(y - yref) <= 1e-9 * babs + 1e-30)),
                              **T["info"])), flush=True)
        return
    import torch
    lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libpb_probe.so"))
    stage_b, region_b = 4 * int(os.environ.get("PB_C", 8192)) + 12 * int(T["chunks"]["nrun"].max()) + 16, 4 * (T["bins"]["rlen"].max() + 12) + (2 * int(T["bins"]["plen"].max()) + 64 if os.environ.get("PB_POS_SMEM") == "1" else 0)
    assert lib.pb_setup(stage_b, int(region_b)) == 0
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.uint8)).cuda()
    d = {k: dev(T[k]) for k in ("cd", "chunks", "runs", "bins", "slabs", "pos", "rcum", "rid")}
    if hasattr(lib, "pb_set_rid"):
        assert lib.pb_set_rid(ctypes.c_void_p(d["rid"].data_ptr())) == 0
    dv = torch.from_numpy(val_o1).cuda() if val_o1 is not None else None
    xt = torch.from_numpy(x).cuda()
    stride = (T["info"]["max_group_entries"] + 16 + 63) // 64 * 64
    buf = torch.empty(2 * stride, device="cuda")
    overlap = os.environ.get("PB_OVERLAP", "0") == "1"
    yt = torch.full((Gr.n,), float("nan"), device="cuda")
    gc = (ctypes.c_int32 * len(T["gc"]))(*T["gc"].tolist())
    gb = (ctypes.c_int32 * len(T["gb"]))(*T["gb"].tolist())
    vp = lambda t: ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)
    stream = torch.cuda.current_stream().cuda_stream

    def run(phases=None):
        phases = phases if phases is not None else ((8 if os.environ.get("PB_PIPE") == "1" else 4) if overlap else 3)
        rc = lib.pb_run(G, phases, gc, gb, vp(d["chunks"]), vp(d["runs"]), vp(d["cd"]), vp(dv), vp(xt), vp(buf),
                        vp(d["bins"]), vp(d["slabs"]), vp(d["pos"]), vp(d["rcum"]), vp(yt), stage_b, int(region_b),
                        ctypes.c_void_p(stream), ctypes.c_longlong(stride))
        assert rc == 0, rc
    run()
    torch.cuda.synchronize()
    y = yt.cpu().numpy().astype(np.float64)
    ok = bool(np.all(np.abs(y - yref) <= 1e-5 * babs + 1e-30))
    y0 = yt.clone()
    for _ in range(5):
        run()
    torch.cuda.synchronize()
    det = bool(torch.equal(y0, yt))
    res = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50):
            run()
        e1.record()
        torch.cuda.synchronize()
        res.append(e0.elapsed_time(e1) * 1000 / 50)
    us = float(np.median(res))
    ph = {}
    for mask in (1, 2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            run(mask)
        e1.record()
        torch.cuda.synchronize()
        ph["expand_us" if mask == 1 else "reduce_us"] = round(e0.elapsed_time(e1) * 1000 / 20, 1)
    m = T["info"]["m"]
    print(json.dumps(dict(cfg=cfg, pattern=pattern, overlap=overlap, ok=ok, deterministic=det, us=round(us, 1), **ph,
                          gflops=round(2 * m / us / 1e3, 1),
                          alg_GBps=round(((4 if pattern else 8) * m + 12 * Gr.n) / us / 1e3, 1),
                          static_bytes_per_nnz=round((4 * m + (0 if pattern else 4 * m) + 2 * T["info"]["npos"]) / m, 2),
                          **T["info"])), flush=True)


if __name__ == "__main__":
    main()
