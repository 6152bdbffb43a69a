"""Row-partitioned solver path (Sec. 3.2) on one GPU: world = 1 runs every step of the multi-GPU
iteration (local plan over the owned rows, epilogue into the allgather slot, fp64 partials in the
slot, rank-order finalize, x permutation from the gathered buffer) except the NCCL call itself.
Parity with the fp64 oracle at the same iteration count (reading R14)."""
import numpy as np
import pytest

import graphgen
import oracle

pytestmark = pytest.mark.gpu


def comm1():
    from paper_1103_2405_b200 import Comm
    return Comm(0, 1, b"\0" * 128, 0)


@pytest.mark.parametrize("cfg", ["t_small", "t_mid"])
def test_dist_pagerank_world1(cfg, gpu):
    from paper_1103_2405_b200 import Solver
    G = graphgen.make_graph(cfg)
    c = comm1()
    s = Solver("pagerank", G.n, G.row_ptr, G.col, device=0, comm=c)
    info = s.run()
    p = s.result().astype(np.float64)
    ref, r = oracle.pagerank(G.n, G.row_ptr, G.col, fixed_iters=info["iterations"])
    assert np.abs(p - ref).sum() < 1e-6, info
    # same iterate as the single-GPU solver path (different plans: tolerance, not bits)
    s1 = Solver("pagerank", G.n, G.row_ptr, G.col, device=0, two_phase=0)
    i1 = s1.run()
    assert abs(i1["iterations"] - info["iterations"]) <= 1


def test_dist_rwr_world1(gpu):
    from paper_1103_2405_b200 import Solver
    G = graphgen.make_graph("t_small")
    s = Solver("rwr", G.n, G.row_ptr, G.col, device=0, comm=comm1())
    q = int(np.nonzero(np.diff(G.row_ptr) > 0)[0][3])
    info = s.run(q)
    r = s.result().astype(np.float64)
    ref, _ = oracle.rwr(G.n, G.row_ptr, G.col, q, fixed_iters=info["iterations"])
    assert np.abs(r - ref).sum() < 1e-6, info


@pytest.mark.parametrize("norm", [1, 2])
def test_dist_hits_world1(norm, gpu):
    from paper_1103_2405_b200 import Solver
    G = graphgen.make_graph("t_small")
    s = Solver("hits", G.n, G.row_ptr, G.col, device=0, comm=comm1(), iter_kw=dict(hits_norm=norm))
    info = s.run()
    a, h = s.result()
    ra, rh, _ = oracle.hits(G.n, G.row_ptr, G.col, norm=norm, fixed_iters=info["iterations"])
    bar_a = 1e-6 * (1.0 if norm == 1 else np.abs(ra).sum())
    bar_h = 1e-6 * (1.0 if norm == 1 else np.abs(rh).sum())
    assert np.abs(a - ra).sum() < bar_a and np.abs(h - rh).sum() < bar_h, info
    # the same number of normalisations as the single-GPU solver on the same (one-pass) kernel:
    # unit-L2 halves stop on fp32 noise near tol (R3), so a different summation order
    # (two-phase tiles) can move the stop by several iterations
    s1 = Solver("hits", G.n, G.row_ptr, G.col, device=0, iter_kw=dict(hits_norm=norm), two_phase=0)
    assert abs(s1.run()["iterations"] - info["iterations"]) <= 1


@pytest.mark.parametrize("algo", ["pagerank", "rwr", "hits"])
def test_dist_needed_exchange_world1(algo, gpu):
    """exchange = 1 (needed columns): own-slot indexing, the partial-offset table
    and the rank-order finalize on one GPU; parity with the oracle at the same iteration count."""
    from paper_1103_2405_b200 import Solver
    G = graphgen.make_graph("t_small")
    s = Solver(algo, G.n, G.row_ptr, G.col, device=0, comm=comm1(), iter_kw=dict(exchange=1))
    q = int(np.nonzero(np.diff(G.row_ptr) > 0)[0][3])
    info = s.run(q) if algo == "rwr" else s.run()
    if algo == "pagerank":
        ref, _ = oracle.pagerank(G.n, G.row_ptr, G.col, fixed_iters=info["iterations"])
        assert np.abs(s.result().astype(np.float64) - ref).sum() < 1e-6, info
    elif algo == "rwr":
        ref, _ = oracle.rwr(G.n, G.row_ptr, G.col, q, fixed_iters=info["iterations"])
        assert np.abs(s.result().astype(np.float64) - ref).sum() < 1e-6, info
    else:
        a, h = s.result()
        ra, rh, _ = oracle.hits(G.n, G.row_ptr, G.col, norm=1, fixed_iters=info["iterations"])
        assert np.abs(a - ra).sum() < 1e-6 and np.abs(h - rh).sum() < 1e-6, info


def _sym_rows(G):
    """rows of A u A^T (RWR's graph, reading R8) as CSR over all vertices."""
    u = (G.keys >> np.uint64(32)).astype(np.int64)
    v = (G.keys & np.uint64(0xFFFFFFFF)).astype(np.int64)
    a = np.concatenate([u, v])
    b = np.concatenate([v, u])
    key = np.unique(a * G.n + b)
    a, b = key // G.n, key % G.n
    rp = np.concatenate([[0], np.cumsum(np.bincount(a, minlength=G.n))]).astype(np.int64)
    return rp, b.astype(np.int32)


@pytest.mark.parametrize("algo", ["pagerank", "rwr"])
def test_local_input_world1(algo, gpu):
    """spmv_solver_create_local (SURVEY 8(b) "*_local"): the rank passes only its rows (here all,
    in a shuffled order) of the iteration matrix with global ids; parity with the oracle."""
    from paper_1103_2405_b200 import Solver
    G = graphgen.make_graph("t_small")
    if algo == "pagerank":
        rp, col = graphgen.keys_to_csr(G.keys, G.n, transpose=True)     # in-neighbours
        deg = np.diff(G.row_ptr).astype(np.int32)
    else:
        rp, col = _sym_rows(G)
        deg = None
    order = np.random.default_rng(3).permutation(G.n).astype(np.int32)
    lens = np.diff(rp)[order]
    lrp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    lcol = np.concatenate([col[rp[v]:rp[v + 1]] for v in order]).astype(np.int32)
    s = Solver.local(algo, G.n, order, lrp, lcol, out_degree=None if deg is None else deg[order],
                     device=0, comm=comm1())
    q = int(np.nonzero(np.diff(G.row_ptr) > 0)[0][3])
    info = s.run(q) if algo == "rwr" else s.run()
    if algo == "pagerank":
        ref, _ = oracle.pagerank(G.n, G.row_ptr, G.col, fixed_iters=info["iterations"])
    else:
        ref, _ = oracle.rwr(G.n, G.row_ptr, G.col, q, fixed_iters=info["iterations"])
    assert np.abs(s.result().astype(np.float64) - ref).sum() < 1e-6, info


def test_local_input_errors(gpu):
    from paper_1103_2405_b200 import Solver, SpmvError
    G = graphgen.make_graph("t_small")
    rp, col = graphgen.keys_to_csr(G.keys, G.n, transpose=True)
    ids = np.arange(G.n, dtype=np.int32)
    with pytest.raises(SpmvError):                     # PageRank without degrees
        Solver.local("pagerank", G.n, ids, rp, col, device=0, comm=comm1())
    with pytest.raises(SpmvError):                     # HITS: block rows n..2n-1 owned by nobody
        Solver.local("hits", G.n, ids, rp, col, device=0, comm=comm1())
    ids2 = np.arange(2 * G.n, dtype=np.int32)
    rp2 = np.concatenate([rp, np.full(G.n, rp[-1])]).astype(np.int64)
    with pytest.raises(SpmvError):                     # HITS takes no out_degree
        Solver.local("hits", G.n, ids2, rp2, col, out_degree=np.ones(2 * G.n, np.int32), device=0, comm=comm1())
    with pytest.raises(SpmvError):                     # a vertex owned by nobody
        Solver.local("rwr", G.n, ids[:-1], rp[:-1], col[:rp[-2]], device=0, comm=comm1())
