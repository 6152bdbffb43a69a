"""Pins for the oracle (-m "not gpu"): the oracle is checked against what the paper and the
mathematics fix -- closed forms, dense solves, SVD, brute force, the paper's worked example --
never against itself.  DESIGN.md "Oracle pins" lists which pin guards which part."""
import json
import math
import os

import numpy as np
import pytest

import graphgen
import oracle
from oracle import format_ref, model_ref, partition_ref

GOLD = os.path.join(os.path.dirname(__file__), "golden")


# ----------------------------------------------------------------------------- helpers
def csr_from_edges(n, edges):
    edges = sorted(set(edges))
    rp = np.zeros(n + 1, dtype=np.int64)
    for u, _ in edges:
        rp[u + 1] += 1
    rp = np.cumsum(rp)
    col = np.array([v for _, v in edges], dtype=np.int32)
    return rp, col


def dense_from_csr(n_rows, n_cols, rp, col, val):
    A = np.zeros((n_rows, n_cols))
    for i in range(n_rows):
        for k in range(rp[i], rp[i + 1]):
            A[i, col[k]] += 1.0 if val is None else float(val[k])
    return A


def random_graph(n, p, seed):
    rng = np.random.default_rng(seed)
    edges = [(u, v) for u in range(n) for v in range(n) if u != v and rng.random() < p]
    return csr_from_edges(n, edges)


# ----------------------------------------------------------------------------- O1 SpMV
def test_spmv_swap_example():
    # [[0,1],[1,0]] . [3,4] = [4,3]
    rp, col = np.array([0, 1, 2]), np.array([1, 0])
    y, b = oracle.spmv(rp, col, np.array([1, 1], np.float32), np.array([3, 4], np.float32))
    assert y.tolist() == [4.0, 3.0] and b.tolist() == [4.0, 3.0]


def test_spmv_identity_and_permutation_exact():
    n = 37
    rng = np.random.default_rng(0)
    x = rng.uniform(-1, 1, n).astype(np.float32)
    y, _ = oracle.spmv(np.arange(n + 1), np.arange(n, dtype=np.int32), np.ones(n, np.float32), x)
    assert np.array_equal(y, x.astype(np.float64))
    perm = rng.permutation(n).astype(np.int32)
    y, _ = oracle.spmv(np.arange(n + 1), perm, None, x)
    assert np.array_equal(y, x[perm].astype(np.float64))


@pytest.mark.parametrize("seed", range(6))
def test_spmv_dense_brute_force(seed):
    rng = np.random.default_rng(seed)
    nr, nc = int(rng.integers(1, 65)), int(rng.integers(1, 65))
    rp, col, val = graphgen.random_csr(nr, nc, int(rng.integers(0, 400)), seed=seed, signed=True)
    x = rng.uniform(-1, 1, nc).astype(np.float32)
    A = dense_from_csr(nr, nc, rp, col, val)
    y, b = oracle.spmv(rp, col, val, x)
    ref = A @ x.astype(np.float64)
    assert np.allclose(y, ref, rtol=0, atol=1e-12)
    absref = np.zeros(nr)
    for i in range(nr):
        for k in range(rp[i], rp[i + 1]):
            absref[i] += abs(float(val[k]) * float(x[col[k]]))
    assert np.allclose(b, absref, rtol=1e-14, atol=0)
    yp, _ = oracle.spmv(rp, col, None, x)          # pattern mode == all-ones values
    Ap = dense_from_csr(nr, nc, rp, col, None)
    assert np.allclose(yp, Ap @ x.astype(np.float64), atol=1e-12)


def test_spmv_one_full_row_vs_fsum():
    n = 20000
    x = graphgen.uniform_f32(n, seed=11, mode=2)
    val = graphgen.uniform_f32(n, seed=12, mode=2)
    y, b = oracle.spmv(np.array([0, n]), np.arange(n, dtype=np.int32), val, x)
    exact = math.fsum(float(v) * float(xx) for v, xx in zip(val, x))
    # left-to-right fp64: |err| <= n * 2^-53 * sum|terms|
    assert abs(y[0] - exact) <= n * 2.0 ** -53 * b[0]


def test_spmv_empty():
    y, b = oracle.spmv(np.zeros(4, np.int64), np.zeros(0, np.int32), np.zeros(0, np.float32),
                       np.ones(5, np.float32))
    assert y.tolist() == [0, 0, 0] and b.tolist() == [0, 0, 0]


# ----------------------------------------------------------------------------- O3 PageRank
def pagerank_dense(n, rp, col, c):
    """(I - c M) p = (1-c)/n 1, M = W^T + (1/n) 1 d^T (d = dangling indicator)."""
    A = dense_from_csr(n, n, rp, col, None)
    od = A.sum(1)
    W = np.zeros_like(A)
    W[od > 0] = A[od > 0] / od[od > 0, None]
    d = (od == 0).astype(float)
    M = W.T + np.outer(np.ones(n), d) / n
    return np.linalg.solve(np.eye(n) - c * M, (1 - c) / n * np.ones(n))


@pytest.mark.parametrize("seed", range(5))
def test_pagerank_dense_solve(seed):
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(2, 65))
    rp, col = random_graph(n, float(rng.uniform(0.02, 0.3)), seed)
    p, r = oracle.pagerank(n, rp, col, c=0.85, tol=1e-14, max_iter=5000)
    ref = pagerank_dense(n, rp, col, 0.85)
    assert r.converged
    assert np.abs(p - ref).sum() < 1e-11
    assert abs(p.sum() - 1.0) < 1e-12


def test_pagerank_cycle_uniform_after_one_iteration():
    n = 9
    rp, col = csr_from_edges(n, [(i, (i + 1) % n) for i in range(n)])
    p, r = oracle.pagerank(n, rp, col, fixed_iters=1)
    assert np.allclose(p, 1.0 / n, atol=1e-16, rtol=0)


@pytest.mark.parametrize("k", [1, 3, 10])
def test_pagerank_in_star_closed_form(k):
    n, c = k + 1, 0.85                       # leaves 1..k -> centre 0 (centre dangling)
    rp, col = csr_from_edges(n, [(i, 0) for i in range(1, n)])
    p, r = oracle.pagerank(n, rp, col, c=c, tol=1e-15, max_iter=10000)
    centre = (c * n + 1 - c) / (n + c * n - c)
    assert abs(p[0] - centre) < 1e-12
    assert np.allclose(p[1:], (1 - centre) / k, atol=1e-12)


@pytest.mark.parametrize("k", [1, 4, 12])
def test_pagerank_out_star_closed_form(k):
    n, c = k + 1, 0.85                       # centre 0 -> leaves (leaves dangling)
    rp, col = csr_from_edges(n, [(0, i) for i in range(1, n)])
    p, r = oracle.pagerank(n, rp, col, c=c, tol=1e-15, max_iter=10000)
    assert abs(p[0] - 1.0 / (n + c)) < 1e-12
    assert np.allclose(p[1:], (k + c) / (k * (n + c)), atol=1e-12)


def test_pagerank_c0_and_two_cycle():
    # SPEC.md L415-L416
    rp, col = random_graph(12, 0.2, 3)
    p, r = oracle.pagerank(12, rp, col, c=0.0, fixed_iters=1)
    assert np.allclose(p, 1 / 12, atol=1e-17)
    rp, col = csr_from_edges(2, [(0, 1), (1, 0)])
    p, r = oracle.pagerank(2, rp, col)
    assert np.allclose(p, [0.5, 0.5], atol=1e-15)


def test_pagerank_mass_invariant_every_iteration():
    G = graphgen.make_graph("t_small")
    for k in (1, 2, 5, 17):
        p, _ = oracle.pagerank(G.n, G.row_ptr, G.col, fixed_iters=k)
        assert abs(p.sum() - 1) < 1e-12 and (p > 0).all()


# ----------------------------------------------------------------------------- O4 HITS
@pytest.mark.parametrize("seed", range(5))
def test_hits_svd(seed):
    rng = np.random.default_rng(200 + seed)
    n = int(rng.integers(3, 65))
    rp, col = random_graph(n, float(rng.uniform(0.1, 0.4)), seed + 50)
    A = dense_from_csr(n, n, rp, col, None)
    U, S, Vt = np.linalg.svd(A)
    if S[0] - S[1] < 1e-3 * S[0]:
        pytest.skip("repeated top singular value: HITS not unique (R28)")
    a, h, r = oracle.hits(n, rp, col, tol=1e-14, max_iter=20000)
    v1, u1 = np.abs(Vt[0]), np.abs(U[:, 0])
    assert np.abs(a - v1).max() < 1e-9 and np.abs(h - u1).max() < 1e-9
    assert abs(np.linalg.norm(a) - 1) < 1e-12 and abs(np.linalg.norm(h) - 1) < 1e-12


def test_hits_star_and_bipartite():
    k = 7
    n = k + 1
    rp, col = csr_from_edges(n, [(i, 0) for i in range(1, n)])
    a, h, r = oracle.hits(n, rp, col, tol=1e-15)
    assert abs(a[0] - 1) < 1e-12 and np.allclose(a[1:], 0, atol=1e-12)
    assert abs(h[0]) < 1e-12 and np.allclose(h[1:], 1 / math.sqrt(k), atol=1e-12)
    S, T = [0, 1, 2], [3, 4, 5, 6]
    rp, col = csr_from_edges(7, [(s, t) for s in S for t in T])
    a, h, r = oracle.hits(7, rp, col, tol=1e-15)
    assert np.allclose(a[T], 0.5, atol=1e-12) and np.allclose(a[S], 0, atol=1e-12)
    assert np.allclose(h[S], 1 / math.sqrt(3), atol=1e-12) and np.allclose(h[T], 0, atol=1e-12)
    a1, h1, _ = oracle.hits(7, rp, col, norm=1, tol=1e-15)    # paper mode: halves sum to 1
    assert np.allclose(a1[T], 0.25) and np.allclose(h1[S], 1 / 3)


def test_hits_empty_graph_uniform():
    a, h, r = oracle.hits(5, np.zeros(6, np.int64), np.zeros(0, np.int32), fixed_iters=3)
    assert np.allclose(a, 1 / math.sqrt(5)) and np.allclose(h, 1 / math.sqrt(5))


# ----------------------------------------------------------------------------- O5 RWR
def rwr_dense(n, rp, col, q, c):
    A = dense_from_csr(n, n, rp, col, None)
    S = ((A + A.T) > 0).astype(float)
    np.fill_diagonal(S, np.diag(A) > 0)
    deg = S.sum(0)
    W = np.zeros_like(S)
    W[:, deg > 0] = S[:, deg > 0] / deg[deg > 0]
    e = np.zeros(n)
    e[q] = 1
    return (1 - c) * np.linalg.solve(np.eye(n) - c * W, e)


@pytest.mark.parametrize("seed", range(5))
def test_rwr_dense_solve(seed):
    rng = np.random.default_rng(300 + seed)
    n = int(rng.integers(2, 65))
    rp, col = random_graph(n, float(rng.uniform(0.03, 0.3)), seed + 90)
    q = int(rng.integers(0, n))
    r, res = oracle.rwr(n, rp, col, q, c=0.9, tol=1e-14, max_iter=20000)
    assert np.abs(r - rwr_dense(n, rp, col, q, 0.9)).sum() < 1e-10


def test_rwr_two_nodes_and_c0():
    rp, col = csr_from_edges(2, [(0, 1)])
    r, _ = oracle.rwr(2, rp, col, 0, c=0.9, tol=1e-15, max_iter=10000)
    assert abs(r[0] - 1 / 1.9) < 1e-12 and abs(r[1] - 0.9 / 1.9) < 1e-12   # 0.526316, 0.473684
    rp, col = random_graph(10, 0.3, 4)
    r, _ = oracle.rwr(10, rp, col, 3, c=0.0, fixed_iters=1)
    assert r[3] == 1.0 and r.sum() == 1.0


def test_rwr_mass_without_isolated():
    n = 30
    rp, col = csr_from_edges(n, [(i, (i + 1) % n) for i in range(n)] + [(0, 15), (7, 22)])
    r, _ = oracle.rwr(n, rp, col, 5, tol=1e-14, max_iter=10000)
    assert abs(r.sum() - 1) < 1e-12


# ----------------------------------------------------------------------------- O6 partition
def test_bitonic_spec_example():
    owner = partition_ref.bitonic_partition([9, 7, 5, 4, 3, 1], 2)
    lens = [9, 7, 5, 4, 3, 1]
    assert sorted(lens[i] for i in range(6) if owner[i] == 0) == [3, 4, 9]
    assert sorted(lens[i] for i in range(6) if owner[i] == 1) == [1, 5, 7]


@pytest.mark.parametrize("P", [1, 2, 3, 5, 8])
def test_bitonic_balance(P):
    rng = np.random.default_rng(P)
    lens = rng.zipf(2.0, 1001)
    owner = np.array(partition_ref.bitonic_partition(lens, P))
    counts = np.bincount(owner, minlength=P)
    assert counts.max() - counts.min() <= 1
    # snake: at every full round the recipient of the longest row alternates ends
    order = sorted(range(1001), key=lambda i: (-lens[i], i))
    assert owner[order[0]] == 0
    if P > 1 and len(order) > P:
        assert owner[order[P]] == P - 1


# ----------------------------------------------------------------------------- O2 format
def fig1():
    with open(os.path.join(GOLD, "fig1.json")) as f:
        g = json.load(f)
    n = g["n_rows"]
    ents = sorted(map(tuple, g["entries_row_col"]))
    rp = np.zeros(n + 1, np.int64)
    for r, _ in ents:
        rp[r + 1] += 1
    rp = np.cumsum(rp)
    col = np.array([c for _, c in ents], np.int32)
    return g, rp, col


def test_fig1_worked_example():
    g, rp, col = fig1()
    ex = g["expected"]
    collen, perm, inv = format_ref.column_order(g["n_cols"], col)
    assert perm.tolist() == ex["column_order"]
    assert int((collen >= 2).sum()) == ex["dense_columns"]
    T = format_ref.paper_tile_count(collen[perm], g["n_cols"], g["tile_width"])
    assert T == ex["num_tiles_alg1"]
    assert model_ref.tile_count(collen[perm], g["n_cols"], g["tile_width"]) == T
    W = g["workload_size"]
    L = format_ref.build(g["n_rows"], g["n_cols"], rp, col, None, g["tile_width"], T, [W] * (T + 1),
                         align_rm=g["warp_size"], ell_h=g["warp_size"])
    t0 = range(L.tiles[0, 2], L.tiles[0, 3])
    got = []
    for j in t0:
        kind = {0: "row_major", 1: "column_major"}[int(L.desc["kind"][j])]
        rb, h = int(L.desc["row_base"][j]), int(L.desc["h"][j])
        rows = [int(r) & (format_ref.FLAG_ACC - 1) for r in L.row_id[rb:rb + h]]
        got.append({"kind": kind, "w": int(L.desc["w"][j]), "h": h, "rows": rows})
    assert got == ex["tile0_workloads"]
    # ranked in-tile lengths of tile 0 (Solution 3 ranking)
    lens = []
    for w in got:
        lens += [w["w"]] * w["h"] if w["kind"] == "row_major" else [w["w"]] * w["h"]
    assert lens == ex["tile0_row_lengths_ranked"]


def test_spec_column_and_row_order_examples():
    # column lengths [1,3,2] -> order [1,2,0]
    _, perm, _ = format_ref.column_order(3, np.array([0, 1, 1, 1, 2, 2], np.int32))
    assert perm.tolist() == [1, 2, 0]
    # Alg. 1 hand traces
    assert format_ref.paper_tile_count(np.array([3, 2, 2, 1, 1]), 5, 2) == 2
    assert format_ref.paper_tile_count(np.array([1, 1, 1, 1]), 4, 2) == 0
    assert format_ref.paper_tile_count(np.array([5, 4, 3, 3, 2, 2, 2, 2]), 8, 2) == 4
    # in-tile row lengths {r0:1, r1:3, r2:2} -> order [r1, r2, r0]
    rp = np.array([0, 1, 4, 6])
    col = np.array([0, 0, 1, 2, 1, 2], np.int32)
    L = format_ref.build(3, 3, rp, col, None, 3, 1, [100, 100], ell_h=32)
    first_rows = [int(r) & (format_ref.FLAG_ACC - 1) for r in L.row_id[:3]]
    assert first_rows == [1, 2, 0]


def test_spec_single_long_row_rm_padding():
    # single row of length 5, warp 32, WL 5 -> one row-major workload w=32, h=1
    L = format_ref.build(1, 5, np.array([0, 5]), np.arange(5, dtype=np.int32), None, 5, 1, [5, 5],
                         align_rm=32)
    assert L.desc["kind"].tolist()[:1] == [0] and L.desc["w"][0] == 32 and L.desc["h"][0] == 1


def test_camping_pad_rule():
    # padded size 512 -> 64 pad slots, next offset 576; 513 -> none
    n = 512
    rp = np.array([0, n])
    L = format_ref.build(1, n, rp, np.arange(n, dtype=np.int32), None, n, 0, [n], align_rm=8,
                         camping_pad=True)
    assert len(L.slot_col) == 576
    rp2 = np.array([0, n, 2 * n])
    L2 = format_ref.build(2, n, rp2, np.concatenate([np.arange(n), np.arange(n)]).astype(np.int32),
                          None, n, 0, [n], align_rm=8, camping_pad=True)
    assert L2.desc["off"].tolist() == [0, 576]
    L3 = format_ref.build(1, 513, np.array([0, 513]), np.arange(513, dtype=np.int32), None, 513, 0,
                          [513], align_rm=1, camping_pad=True)
    assert len(L3.slot_col) == 513


def multiset(rows, cols, vals):
    return sorted(zip(rows.tolist(), cols.tolist(), vals.tolist()))


@pytest.mark.parametrize("seed", range(8))
def test_format_roundtrip_random(seed):
    rng = np.random.default_rng(seed)
    nr, nc = int(rng.integers(1, 300)), int(rng.integers(1, 300))
    kind = "powerlaw" if seed % 2 else "uniform"
    rp, col, val = graphgen.random_csr(nr, nc, int(rng.integers(0, 3000)), seed=seed, kind=kind)
    tw = int(rng.integers(1, 40))
    collen, perm, inv = format_ref.column_order(nc, col)
    T = min(format_ref.paper_tile_count(collen[perm], nc, tw), 3)
    wls = [int(rng.integers(1, 200)) for _ in range(T + 1)]
    L = format_ref.build(nr, nc, rp, col, val, tw, T, wls, align_rm=8,
                         split_long_rows=bool(seed % 3), camping_pad=bool(seed % 4 == 1))
    r, c, v = format_ref.decode_to_coo(L)
    ref_r = np.repeat(np.arange(nr), np.diff(rp))
    assert multiset(r, c, v) == multiset(ref_r, col.astype(np.int64), val.astype(np.float64))
    # every row written exactly once as FINAL, never ACC in its first tile
    fin = np.zeros(nr, int)
    for e in L.row_id.tolist():
        if e != format_ref.PAD_ROW and e & format_ref.FLAG_FINAL:
            fin[e & (format_ref.FLAG_ACC - 1)] += 1
    split_rows = {int(s[0]) & (format_ref.FLAG_ACC - 1): int(s[1]) for s in L.split}
    for i in range(nr):
        assert fin[i] == split_rows.get(i, 1) or (i in split_rows and fin[i] >= 1)
    # shape law (Solution 3): row-major <=> w >= h before padding
    for j in range(len(L.desc["off"])):
        if L.desc["kind"][j] == format_ref.KIND_RM:
            assert L.desc["w"][j] % 8 == 0
        if L.desc["kind"][j] == format_ref.KIND_CM:
            assert L.desc["h"][j] % 32 == 0


def test_format_bruteforce_tiny():
    """every 0/1 pattern of a 3x3 matrix, three parameter sets: decode == input."""
    for mask in range(512):
        ents = [(i // 3, i % 3) for i in range(9) if mask >> i & 1]
        rp = np.zeros(4, np.int64)
        for r, _ in ents:
            rp[r + 1] += 1
        rp = np.cumsum(rp)
        col = np.array([c for _, c in ents], np.int32)
        val = (np.arange(len(ents)) + 1).astype(np.float32)
        for tw, T, wl in ((1, 2, [1, 2, 3]), (2, 1, [2, 1]), (3, 0, [4])):
            collen, perm, _ = format_ref.column_order(3, col)
            T_ok = min(T, format_ref.paper_tile_count(collen[perm], 3, tw))
            L = format_ref.build(3, 3, rp, col, val, tw, T_ok, wl[:T_ok + 1], align_rm=4, ell_h=2)
            r, c, v = format_ref.decode_to_coo(L)
            ref = multiset(np.repeat(np.arange(3), np.diff(rp)), col.astype(np.int64), val.astype(np.float64))
            assert multiset(r, c, v) == ref


# ----------------------------------------------------------------------------- O7 model
def test_eq1_anchor():
    # PAPER.md L124 (960 warps on Tesla) with Eq. 1: ceil(2000/960) = 3
    tot, d = model_ref.pm_paper([1] * 2000, 1, lambda w, h: 1.0, 960)
    assert d["n_warp"] == 2000 and d["I"] == 3 and d["waves"] == 3


def test_uniform_table_total_is_padded_size():
    # throughput 1 everywhere -> total = sum of padded w*h
    rows = [70, 40, 33, 10, 9, 3, 3, 2, 1, 1, 1]
    tot, d = model_ref.pm_paper(rows, 70, lambda w, h: 1.0, 960)
    i, ref = 0, 0
    while i < len(rows):
        w = rows[i]; h = 70 // w
        w, h = model_ref.padding(w, h)
        ref += w * h; i += h
    assert tot == ref
    # by hand: 70 -> (96,1); 40 -> (64,1); 33 -> h=2, (64,2) rows {33,10};
    # 9 -> h=7, 9 >= 7 so row major, (32,7) rows {9,3,3,2,1,1,1}
    assert ref == 96 + 64 + 64 * 2 + 32 * 7 == 512


def test_alg2_candidate_set_hand_trace():
    # longest row 100, nnz = 960*500 -> candidates 100, 200, ..., 500
    rows = [100] * 4800
    seen = []
    model_ref.partition(rows, lambda w, h: (seen.append((w, h)) or 1.0), 960)
    tried = sorted({w * 0 + h for w, h in seen})
    # one PM call per candidate; for uniform rows of 100, h = WL // 100 = 1..5 (before padding)
    assert {h for _, h in seen} == {1, 2, 3, 4, 5}
    assert tried == [1, 2, 3, 4, 5]


# --- pm_packed (the B200 reading of Alg. 3) pinned to the paper's pm_paper and by hand ---------
def _hist(rows):
    out = {}
    for r in rows:
        out[r] = out.get(r, 0) + 1
    return sorted(out.items(), key=lambda kv: -kv[0])


def _paper_sizes(rows, WL):
    """Alg. 3 lines 7-15 written out again as a plain list of padded (w, h) shapes."""
    i, out = 0, []
    while i < len(rows):
        w = rows[i]
        h = WL // w
        wp, hp = model_ref.padding(w, h)
        out.append((wp, hp))
        i += hp
    return out


@pytest.mark.parametrize("seed", range(12))
@pytest.mark.parametrize("fill", [False, True])
def test_pm_packed_equals_pm_paper_in_paper_mode(seed, fill):
    """Paper mode (no split, align 32, WL >= longest row): the B200 walk forms the paper's
    workloads.  The only difference is the last workload, which Alg. 3 counts at its
    full padded shape and the format clips to the rows left (reading R13): equal when it is not
    clipped, and with a uniform table the totals differ by exactly the clipped slots."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(5, 400))
    rows = sorted((int(v) for v in rng.zipf(1.7, n) if v < 500), reverse=True) or [1]
    WL = int(rows[0] * rng.integers(1, 4))
    M = int(rng.integers(1, 50))
    if fill:
        # append rows of the last length until the paper's last workload is full (not clipped)
        wp, hp = _paper_sizes(rows, WL)[-1]
        used = sum(h for _, h in _paper_sizes(rows, WL)[:-1])
        rows = rows + [rows[-1]] * (used + hp - len(rows))
    shape_perf = lambda w, h: 1e9 * (1.0 + (w % 7) + 0.5 * (h % 5))   # any shape-dependent table
    paper, _ = model_ref.pm_paper(rows, WL, shape_perf, M)
    packed = model_ref.pm_packed(_hist(rows), WL, lambda k, w, h: shape_perf(w, h), M, align=32, split=False)
    shapes = _paper_sizes(rows, WL)
    wls = model_ref.packed_workloads(_hist(rows), WL, align=32, split=False)
    assert len(wls) == len(shapes)
    # all but the last workload agree shape by shape
    assert [(w, h) for _, w, h, _ in wls[:-1]] == shapes[:-1]
    clipped = sum(w * h for w, h in shapes) - sum(size for *_, size in wls)
    assert clipped >= 0 and (clipped == 0) == fill
    if clipped == 0:
        assert math.isclose(packed, paper, rel_tol=1e-12)
    up, _ = model_ref.pm_paper(rows, WL, lambda w, h: 1e9, M)
    uk = model_ref.pm_packed(_hist(rows), WL, lambda k, w, h: 1e9, M, align=32, split=False)
    assert math.isclose(up - uk, clipped / 1e9, rel_tol=1e-9, abs_tol=1e-18)


def test_pm_packed_clipped_last_slab_hand_trace():
    """Rows [4]*5 + [1]*40, WL 64.  Paper mode: 4 -> h = 16 -> column major, padded (4, 32);
    1 -> h = 64, (1, 64): 128 + 64 = 192 slots.  The format clips the second slab to the 13 rows
    left, padded to 32: 128 + 32 = 160 slots, 32 fewer."""
    rows = [4] * 5 + [1] * 40
    assert model_ref.pm_paper(rows, 64, lambda w, h: 1.0, 960)[0] == 192
    wls = model_ref.packed_workloads(_hist(rows), 64, align=32, split=False)
    assert wls == [("cm", 4, 32, 128), ("cm", 1, 32, 32)]
    # MAX_ACT_WARP 1: one wave per workload, t = Size / P (Eq. 3 with P_i of one warp)
    t = model_ref.pm_packed(_hist(rows), 64, lambda k, w, h: 2e9 if (w, h) == (4, 32) else 1e9, 1,
                            align=32, split=False)
    assert math.isclose(t, 128 / 2e9 + 32 / 1e9, rel_tol=1e-15)


def test_pm_packed_split_row_hand_trace():
    """Rows [70, 9, 9, 3, 2, 2, 1], WL 32, align 8, split (reading R21):
      70 > WL -> chunks 32, 32, 6 -> RM (32,1), (32,1), (8,1);
      9: hq = 3 <= 9 -> RM of 3 rows {9, 9, 3}, width 16 -> 48 slots;
      2: hq = 16 > 2 -> CM, take min(32, 3 rows left) -> slab (2, 32) = 64 slots.
    Sizes 32 + 32 + 8 + 48 + 64 = 184."""
    h = _hist([70, 9, 9, 3, 2, 2, 1])
    wls = model_ref.packed_workloads(h, 32, align=8, split=True)
    assert wls == [("rm", 32, 1, 32), ("rm", 32, 1, 32), ("rm", 8, 1, 8), ("rm", 16, 3, 48), ("cm", 2, 32, 64)]
    # uniform table: total = padded slots / throughput
    assert math.isclose(model_ref.pm_packed(h, 32, lambda k, w, hh: 1e9, 2), 184e-9, rel_tol=1e-15)
    # two-valued table, MAX_ACT_WARP 2: waves {32,32} rm, {8,48} rm, {64} cm at 4e9:
    #   64/1e9 + 56/1e9 + 64/4e9 = 136e-9
    two = lambda k, w, hh: 1e9 if k == "rm" else 4e9
    assert math.isclose(model_ref.pm_packed(h, 32, two, 2), 136e-9, rel_tol=1e-15)
    # MAX_ACT_WARP 3: waves {32,32,8} rm -> 72/1e9; {48 rm, 64 cm} -> mean P 2.5e9 -> 112/2.5e9
    assert math.isclose(model_ref.pm_packed(h, 32, two, 3), 72e-9 + 44.8e-9, rel_tol=1e-15)


def test_tile_time_us_terms_by_hand():
    """The B200 per-launch terms, computed by hand.  Tile 2 of a tiling (y RMW charged), staged
    (cached), 1000 rows of length 1, WL 100: w = 1 < hq = 100 -> column major, take =
    min(rup(100, 32) = 128, rows left): 7 slabs of 128 rows and one of the last 104 rows (padded
    to 128) = 8 workloads of 128 slots."""
    h = [(1, 1000)]
    wls = model_ref.packed_workloads(h, 100)
    assert len(wls) == 8 and all(w == ("cm", 1, 128, 128) for w in wls[:7]) and wls[7] == ("cm", 1, 128, 128)
    # 1000 = 7*128 + 104: the 8th slab takes the last 104 rows (padded to 128): 8 workloads
    us = model_ref.tile_time_us(h, 100, lambda k, w, hh: 1e9, 4, tile_index=2, tile_width=65536, cached=True,
                                launch_us=3.0, stage_GBps=5000.0, rmw_GBps=2500.0, tail_frac=0.5, sm_count=148)
    waves = 8 * 128 / 1e9 * 1e6                                  # 1.024 us (uniform table)
    tail = 0.5 * 100 * 4 / 1e9 * 1e6                             # 0.2 us
    stage = 65536 * 4 * 148 / 5e6                                # 7.759462... us
    rmw = 1000 * 8 / 2.5e6                                       # 3.2 us
    assert math.isclose(us, waves + tail + 3.0 + stage + rmw, rel_tol=1e-12)
    assert math.isclose(stage, 7.7594624, rel_tol=1e-9)
    # first tile, unstaged: no staging, no RMW; an empty tile costs nothing
    us0 = model_ref.tile_time_us(h, 100, lambda k, w, hh: 1e9, 4, tile_index=0, tile_width=65536, cached=False,
                                 launch_us=3.0, stage_GBps=5000.0, rmw_GBps=2500.0)
    assert math.isclose(us0, waves + 3.0, rel_tol=1e-12)
    assert model_ref.tile_time_us([], 100, lambda k, w, hh: 1e9, 4, tile_index=1, tile_width=8, cached=True,
                                  launch_us=3.0, stage_GBps=1.0, rmw_GBps=1.0) == 0.0


def test_b200_candidate_set_by_hand():
    """Reading R21: powers of two from 32 to max(L, 32768) plus the first 96 multiples of the
    longest row L that do not exceed it (table bound)."""
    c = model_ref.b200_candidates(100)
    assert [v for v in c if v & (v - 1) == 0] == [32, 64, 128, 256, 512, 1024, 2048, 4096, 8192, 16384, 32768]
    assert [v for v in c if v % 100 == 0] == [100 * k for k in range(1, 97)]
    assert len(c) == 11 + 96              # no power of two is a multiple of 100 (25 does not divide it)
    c = model_ref.b200_candidates(50000)
    assert c[-1] == 50000 and 32768 in c and 65536 not in c and len(c) == 12


def test_tile_coo_packing_by_hand():
    """TILE-COO workloads (orient 3): rows [70, 9, 9, 3, 2, 2, 1], WL 32, split: the row of 70
    becomes chunks 32, 32, 6 (padded to 8) as in the composite; then whole rows while at most 32
    entries: 9 + 9 + 3 + 2 + 2 + 1 = 26 -> one workload of 26 entries padded to 32 slots.  With
    WL 16: {9} (9 + 9 > 16), {9, 3, 2, 2} = 16, {1} -> 16, 16, 32 slots."""
    h = _hist([70, 9, 9, 3, 2, 2, 1])
    assert model_ref.packed_workloads(h, 32, align=8, split=True, orient=3) == [
        ("rm", 32, 1, 32), ("rm", 32, 1, 32), ("rm", 8, 1, 8), ("rm", 32, 1, 32)]
    assert model_ref.packed_workloads(_hist([9, 9, 3, 2, 2, 1]), 16, orient=3) == [
        ("rm", 32, 1, 32), ("rm", 32, 1, 32), ("rm", 32, 1, 32)]
