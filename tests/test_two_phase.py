"""Two-phase tiles (csrc/pb.h): the layout decodes back to the input entries (CPU,
host-only plans), and the product equals the fp64 oracle within the north-star bar on the GPU,
including several groups, chunks cut by every limit, rows longer than a region and empty rows."""
import numpy as np
import pytest

import graphgen
import oracle

RTOL = 1e-5

# small caps so that tiny matrices still span several groups / chunks / bins / long rows
SMALL = dict(two_phase=1, pb_region=64, pb_chunk=37, pb_xcap=50, pb_group=300)

CASES = [
    # (nr, nc, nnz, kind, valued, signed, options)
    (300, 200, 3000, "uniform", True, False, SMALL),
    (1000, 1000, 20000, "powerlaw", True, True, SMALL),
    (1000, 1000, 20000, "powerlaw", False, False, SMALL),
    (777, 3001, 40000, "powerlaw", True, False, dict(SMALL, pb_region=512, pb_chunk=300, pb_xcap=700)),
    (5000, 300, 60000, "uniform", True, True, dict(two_phase=1, pb_region=128, pb_group=5000)),
    (3000, 3000, 90000, "powerlaw", True, False, dict(two_phase=1)),
    (3000, 3000, 90000, "powerlaw", False, False, dict(two_phase=1, pb_group=20000)),
    (50, 9000, 700, "uniform", True, True, dict(two_phase=1, pb_xcap=1)),
    (9000, 50, 700, "uniform", True, True, dict(two_phase=1, pb_chunk=1)),
]


def _coo_sorted(rp, col, val):
    nr = len(rp) - 1
    v = np.ones(len(col), np.float32) if val is None else val
    return sorted(zip(np.repeat(np.arange(nr), np.diff(rp)).tolist(), col.tolist(), v.tolist()))


@pytest.mark.parametrize("case", range(len(CASES)))
def test_layout_decodes_to_input(case):
    from paper_1103_2405_b200 import Plan
    nr, nc, nnz, kind, valued, signed, opt = CASES[case]
    rp, col, val = graphgen.random_csr(nr, nc, nnz, seed=case, kind=kind, valued=valued, signed=signed)
    p = Plan(nr, nc, rp, col, val, device=-1, **opt)
    st = p.stats()
    assert st["two_phase"] and st["pb_bins"] >= 1 and st["pb_groups"] >= 1
    r, c, v = p.to_coo()
    assert sorted(zip(r.tolist(), c.tolist(), v.tolist())) == _coo_sorted(rp, col, val)


def test_layout_limits_hold():
    """Every chunk respects xcap / ccap, groups respect the group size (one bin may exceed it),
    and a row longer than a region forms a bin of its own."""
    from paper_1103_2405_b200 import Plan
    n = 400
    lens = np.zeros(n, np.int64)
    lens[5] = 1000                                      # > pb_region -> long-row bin
    lens[7:300] = np.random.default_rng(1).integers(0, 30, 293)
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    col = np.concatenate([np.sort(np.random.default_rng(i).choice(2000, l, replace=False)) for i, l in enumerate(lens)]).astype(np.int32)
    p = Plan(n, 2000, rp, col, None, device=-1, **SMALL)
    st = p.stats()
    assert st["pb_long_bins"] == 1
    r, c, _ = p.to_coo()
    assert sorted(zip(r.tolist(), c.tolist())) == sorted(zip(np.repeat(np.arange(n), lens).tolist(), col.tolist()))


def test_empty_and_zero_rows():
    from paper_1103_2405_b200 import Plan
    p = Plan(7, 5, np.zeros(8, np.int64), np.zeros(0, np.int32), np.zeros(0, np.float32), device=-1, two_phase=1)
    r, c, v = p.to_coo()
    assert len(r) == 0 and p.stats()["two_phase"]


def test_model_chooses_by_prediction():
    """two_phase = -1: the plan takes the execution with the smaller predicted time."""
    from paper_1103_2405_b200 import Plan
    rp, col, val = graphgen.random_csr(3000, 3000, 90000, seed=5, kind="powerlaw", valued=True)
    st = Plan(3000, 3000, rp, col, val, device=-1).stats()
    assert st["two_phase"] == (st["two_phase_predicted_us"] < st["one_pass_predicted_us"])
    for forced in (0, 1):
        s2 = Plan(3000, 3000, rp, col, val, device=-1, two_phase=forced).stats()
        assert s2["two_phase"] == bool(forced)


# ----------------------------------------------------------------------------- GPU parity
def _run(nr, nc, rp, col, val, x, **opt):
    import torch
    from paper_1103_2405_b200 import Plan
    p = Plan(nr, nc, rp, col, val, device=0, **opt)
    xt = torch.from_numpy(np.ascontiguousarray(x, np.float32)).cuda()
    yt = torch.full((max(nr, 1),), float("nan"), device="cuda")
    p.execute(xt, yt)
    torch.cuda.synchronize()
    return p, yt.cpu().numpy()[:nr]


def _check(y, rp, col, val, x):
    yref, b = oracle.spmv(rp, col, val, x)
    err = np.abs(y.astype(np.float64) - yref)
    bad = err > RTOL * b + 1e-30
    assert not bad.any(), f"{bad.sum()} rows off; worst {err[bad][:5]} vs bound {(RTOL * b)[bad][:5]}"


@pytest.mark.gpu
@pytest.mark.parametrize("case", range(len(CASES)))
def test_gpu_parity(case, gpu):
    nr, nc, nnz, kind, valued, signed, opt = CASES[case]
    rp, col, val = graphgen.random_csr(nr, nc, nnz, seed=case, kind=kind, valued=valued, signed=signed)
    x = graphgen.uniform_f32(nc, seed=3, mode=2 if signed else 0)
    if not valued:
        opt = dict(opt, pattern=1)
    p, y = _run(nr, nc, rp, col, val, x, **opt)
    assert p.stats()["two_phase"]
    _check(y, rp, col, val, x)


@pytest.mark.gpu
def test_gpu_edge_cases_and_determinism(gpu):
    import torch
    # nnz = 0: every row written as 0
    p, y = _run(7, 5, np.zeros(8, np.int64), np.zeros(0, np.int32), np.zeros(0, np.float32),
                np.ones(5, np.float32), two_phase=1)
    assert (y == 0).all()
    # one full row far longer than a region (long-row bin) beside a short one
    n = 100_003
    rp = np.array([0, n, n + 1])
    col = np.concatenate([np.arange(n), [7]]).astype(np.int32)
    val = graphgen.uniform_f32(n + 1, seed=9, mode=2)
    x = graphgen.uniform_f32(n, seed=10, mode=2)
    p, y = _run(2, n, rp, col, val, x, two_phase=1)
    _check(y, rp, col, val, x)
    assert p.stats()["pb_long_bins"] == 1
    # permutation matrix: exact
    m = 4099
    perm = np.random.default_rng(0).permutation(m).astype(np.int32)
    x = graphgen.uniform_f32(m, seed=11, mode=2)
    p, y = _run(m, m, np.arange(m + 1), perm, np.ones(m, np.float32), x, two_phase=1, pb_xcap=100, pb_group=700)
    assert np.array_equal(y, x[perm])
    # bitwise run to run, repeated launches reuse the queue counters
    G = graphgen.make_graph("t_mid")
    val = graphgen.edge_values(G.keys, seed=graphgen.SEED_VAL, mode=1)
    x = graphgen.uniform_f32(G.n, seed=3)
    from paper_1103_2405_b200 import Plan
    p = Plan(G.n, G.n, G.row_ptr, G.col, val, device=0, two_phase=1, pb_group=200_000)
    assert p.stats()["pb_groups"] >= 4
    xt = torch.from_numpy(x).cuda()
    ys = []
    for _ in range(3):
        yt = torch.empty(G.n, device="cuda")
        p.execute(xt, yt)
        torch.cuda.synchronize()
        ys.append(yt.cpu().numpy())
    assert ys[0].tobytes() == ys[1].tobytes() == ys[2].tobytes()
    _check(ys[0], G.row_ptr, G.col, val, x)
