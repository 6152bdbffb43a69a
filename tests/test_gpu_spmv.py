"""GPU parity of the tiled-composite SpMV (through the C ABI) against the fp64 oracle.
Bar (BASELINE.json north_star): |y - y_ref| <= 1e-5 * sum_j |a_ij x_j| + 1e-30 per element."""
import numpy as np
import pytest

import graphgen
import oracle

pytestmark = pytest.mark.gpu

RTOL = 1e-5


def run_plan(nr, nc, rp, col, val, x, **opt):
    import torch
    from paper_1103_2405_b200 import Plan
    p = Plan(nr, nc, rp, col, val, device=0, **opt)
    xt = torch.from_numpy(np.ascontiguousarray(x, np.float32)).cuda()
    yt = torch.full((max(nr, 1),), float("nan"), device="cuda")
    p.execute(xt, yt)
    torch.cuda.synchronize()
    return p, yt.cpu().numpy()[:nr]


def check(y, rp, col, val, x):
    yref, b = oracle.spmv(rp, col, val, x)
    err = np.abs(y.astype(np.float64) - yref)
    bad = err > RTOL * b + 1e-30
    assert not bad.any(), f"{bad.sum()} rows off; worst {err[bad][:5]} vs bound {(RTOL * b)[bad][:5]}"


CASES = [
    # (nr, nc, nnz, kind, valued, signed, options)
    (300, 200, 3000, "uniform", True, False, dict(tile_width=16, num_tiles=3, workload_size=64)),
    (1000, 1000, 20000, "powerlaw", True, True, dict(tile_width=64, num_tiles=4, workload_size=128)),
    (1000, 1000, 20000, "powerlaw", False, False, dict(tile_width=64, num_tiles=4, workload_size=128)),
    (777, 3001, 40000, "powerlaw", True, False, dict(tile_width=100, num_tiles=2, workload_sizes=[37, 512, 1000])),
    (5000, 300, 60000, "uniform", True, True, dict(tile_width=300, num_tiles=1, workload_size=4096)),
    (2000, 2000, 50000, "powerlaw", True, False, dict(tile_width=512, num_tiles=2, workload_size=96, stage_x=0)),
    (2000, 2000, 50000, "powerlaw", True, False, dict(tile_width=512, num_tiles=2, workload_size=96, align_rm=32)),
    (2000, 2000, 50000, "powerlaw", True, False, dict(tile_width=512, num_tiles=2, workload_size=96, camping_pad=1)),
    (3000, 3000, 90000, "powerlaw", True, False, dict(num_tiles=0, split_long_rows=0)),
    (3000, 3000, 90000, "powerlaw", True, False, dict()),
    # f2 single-format layouts: CSR-vector (row major only) and ELL (column major only)
    (3000, 3000, 90000, "powerlaw", True, True, dict(orient=1)),
    (3000, 3000, 90000, "powerlaw", False, False, dict(orient=1, tile_width=256, num_tiles=2, workload_size=256)),
    (3000, 3000, 90000, "powerlaw", True, True, dict(orient=2)),
    (3000, 3000, 90000, "powerlaw", False, False, dict(orient=2, tile_width=256, num_tiles=2, workload_size=512)),
    # f2 TILE-COO: COO dense tiles (segmented warp sums), composite remainder
    (3000, 3000, 90000, "powerlaw", True, True, dict(orient=3, tile_width=256, num_tiles=3, workload_size=256)),
    (3000, 3000, 90000, "powerlaw", False, False, dict(orient=3, tile_width=64, num_tiles=4, workload_size=40)),
    (2000, 2000, 50000, "powerlaw", True, False, dict(orient=3, tile_width=512, num_tiles=2, workload_size=96, stage_x=0)),
    (1000, 5000, 40000, "uniform", True, True, dict(orient=3, tile_width=1000, num_tiles=4, workload_size=5000,
                                                    split_long_rows=0)),
    # the model's choice among the four
    (3000, 3000, 90000, "powerlaw", True, False, dict(orient=-1)),
]


@pytest.mark.parametrize("case", range(len(CASES)))
def test_spmv_parity_random(case, gpu):
    nr, nc, nnz, kind, valued, signed, opt = CASES[case]
    rp, col, val = graphgen.random_csr(nr, nc, nnz, seed=case, kind=kind, valued=valued, signed=signed)
    x = graphgen.uniform_f32(nc, seed=3, mode=2 if signed else 0)
    if not valued:
        opt = dict(opt, pattern=1)
    p, y = run_plan(nr, nc, rp, col, val, x, **opt)
    check(y, rp, col, val, x)


def test_edge_cases(gpu):
    # nnz = 0 (empty rows are written as 0, never left stale)
    p, y = run_plan(7, 5, np.zeros(8, np.int64), np.zeros(0, np.int32), np.zeros(0, np.float32),
                    np.ones(5, np.float32))
    assert (y == 0).all()
    # 1x1
    p, y = run_plan(1, 1, np.array([0, 1]), np.array([0], np.int32), np.array([2.5], np.float32),
                    np.array([4.0], np.float32))
    assert y.tolist() == [10.0]
    # one full row, far longer than WL: split into chunks, combined in chunk order
    n = 100_003
    rp = np.array([0, n, n + 1])
    col = np.concatenate([np.arange(n), [7]]).astype(np.int32)
    val = graphgen.uniform_f32(n + 1, seed=9, mode=2)
    x = graphgen.uniform_f32(n, seed=10, mode=2)
    p, y = run_plan(2, n, rp, col, val, x, workload_size=1000, tile_width=4096, num_tiles=3)
    check(y, rp, col, val, x)
    assert p.stats()["n_split"] >= 1
    # all rows of length 1, identity and permutation matrices are exact
    m = 4099
    perm = np.random.default_rng(0).permutation(m).astype(np.int32)
    x = graphgen.uniform_f32(m, seed=11, mode=2)
    p, y = run_plan(m, m, np.arange(m + 1), perm, np.ones(m, np.float32), x, tile_width=1024, num_tiles=2)
    assert np.array_equal(y, x[perm])
    # rectangular with empty columns and rows; signed values
    rp, col, val = graphgen.random_csr(50, 9000, 700, seed=4, signed=True)
    x = graphgen.uniform_f32(9000, seed=12, mode=2)
    p, y = run_plan(50, 9000, rp, col, val, x, tile_width=2048, num_tiles=2, workload_size=8)
    check(y, rp, col, val, x)


def test_graph_auto_and_deterministic(gpu):
    import torch
    from paper_1103_2405_b200 import Plan
    G = graphgen.make_graph("t_mid")
    rp, col = graphgen.keys_to_csr(G.keys, G.n, transpose=True)
    val = graphgen.edge_values(G.keys[np.lexsort((G.keys >> np.uint64(32), G.keys & np.uint64(0xFFFFFFFF)))])
    x = graphgen.uniform_f32(G.n, seed=3)
    for opt in (dict(), dict(tile_width=8192, num_tiles=4, workload_size=512)):
        p = Plan(G.n, G.n, rp, col, val, device=0, **opt)
        xt = torch.from_numpy(x).cuda()
        y1 = torch.empty(G.n, device="cuda"); y2 = torch.empty(G.n, device="cuda")
        p.execute(xt, y1); p.execute(xt, y2)
        torch.cuda.synchronize()
        a, b = y1.cpu().numpy(), y2.cpu().numpy()
        assert a.tobytes() == b.tobytes()            # bitwise run-to-run
        check(a, rp, col, val, x)
        yh = p.execute_host(x)                       # host path through the C ABI
        assert yh.tobytes() == a.tobytes()
        # pipelined batch: 5 different x (odd count: both buffer pairs, ragged last round)
        X = np.stack([graphgen.uniform_f32(G.n, seed=30 + b) for b in range(5)])
        Y = p.execute_host_batch(X)
        for b in range(5):
            xt = torch.from_numpy(X[b]).cuda()
            p.execute(xt, y1)
            torch.cuda.synchronize()
            assert Y[b].tobytes() == y1.cpu().numpy().tobytes()
        assert p.execute_host_batch(X[:0]).shape == (0, G.n)


@pytest.mark.parametrize("cfg", ["c2", "c3_flickr", "c3_youtube"])
@pytest.mark.parametrize("two_phase", [-1, 0])
def test_full_size_every_row(cfg, two_phase, gpu):
    """BASELINE configs[1] (c2) and the configs[2] shapes at full size, valued, in the launch
    configuration bench.py times (auto plan: the model's execution) and with the one-pass tiles
    forced: EVERY row against the fp64 oracle (the multi-threaded oracle does the whole product
    in well under a second), then bitwise determinism."""
    import torch
    from paper_1103_2405_b200 import Plan
    G = graphgen.make_graph(cfg)
    val = graphgen.edge_values(G.keys, seed=graphgen.SEED_VAL, mode=1)
    x = graphgen.uniform_f32(G.n, seed=graphgen.SEED_X)
    p = Plan(G.n, G.n, G.row_ptr, G.col, val, device=0, two_phase=two_phase)
    xt = torch.from_numpy(x).cuda()
    yt = torch.empty(G.n, device="cuda")
    p.execute(xt, yt)
    torch.cuda.synchronize()
    y = yt.cpu().numpy()
    yref, b = oracle.spmv(G.row_ptr, G.col, val, x)
    err = np.abs(y.astype(np.float64) - yref)
    bad = err > RTOL * b + 1e-30
    assert not bad.any(), f"{bad.sum()} of {G.n} rows off"
    y2 = torch.empty(G.n, device="cuda")
    p.execute(xt, y2)
    assert y2.cpu().numpy().tobytes() == y.tobytes()


@pytest.mark.parametrize("shape", [(2048, 2048), (300, 5000), (5000, 40)])
def test_dense_matrices(shape, gpu):
    """Appendix D dense case (§8(f) f4): every row is full; rows longer than WL split."""
    nr, nc = shape
    rp, col, val = graphgen.dense_csr(nr, nc)
    x = graphgen.uniform_f32(nc, seed=graphgen.SEED_X)
    _, y = run_plan(nr, nc, rp, col, val, x)
    check(y, rp, col, val, x)


@pytest.mark.parametrize("half_band,drop", [(13, 0.0), (4, 0.3), (40, 0.5)])
def test_banded_matrices(half_band, drop, gpu):
    """FEM-like banded matrices (§8(f) f4), with and without a ragged band."""
    n = 50_000
    rp, col, val = graphgen.banded_csr(n, half_band, drop=drop)
    x = graphgen.uniform_f32(n, seed=graphgen.SEED_X, mode=2)
    _, y = run_plan(n, n, rp, col, val, x)
    check(y, rp, col, val, x)


def test_permute_scatter_equals_gather(gpu, monkeypatch):
    """a7: the gather form x'[k] = x[perm[k]] (default) and the scatter form x'[inv[j]] = x[j]
    (TCSPMV_PERMUTE=scatter) build the same x', so the products are bitwise equal; odd n_cols
    exercises the vector body and the scalar tail."""
    import torch
    from paper_1103_2405_b200 import Plan
    rp, col, val = graphgen.random_csr(3001, 4099, 60000, seed=5, kind="powerlaw", valued=True)
    x = torch.from_numpy(graphgen.uniform_f32(4099, seed=3)).cuda()
    out = []
    for mode in (None, "scatter"):
        if mode:
            monkeypatch.setenv("TCSPMV_PERMUTE", mode)
        p = Plan(3001, 4099, rp, col, val, device=0)
        y = torch.empty(3001, device="cuda")
        p.execute(x, y)
        torch.cuda.synchronize()
        out.append(y.cpu().numpy())
        p.close()
    assert out[0].tobytes() == out[1].tobytes()
    check(out[0], rp, col, val, x.cpu().numpy())


def test_plain_c_consumer_on_gpu(gpu, tmp_path):
    """The whole path through the C ABI from a C99 program (no Python/torch on the path): valued
    SpMV via spmv_execute_host and the one-shot pagerank(), checked against the fp64 oracle."""
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    libdir = os.path.join(root, "paper_1103_2405_b200", "lib")
    exe = str(tmp_path / "abi_gpu_consumer")
    r = subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(root, "include"),
                        os.path.join(root, "tests", "c", "abi_gpu_consumer.c"), "-L", libdir, "-ltcspmv",
                        "-Wl,-rpath," + libdir, "-o", exe], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    G = graphgen.make_graph("t_mid")
    rp, col = graphgen.keys_to_csr(G.keys, G.n, transpose=True)
    val = graphgen.edge_values(G.keys[np.lexsort((G.keys >> np.uint64(32), G.keys & np.uint64(0xFFFFFFFF)))])
    x = graphgen.uniform_f32(G.n, seed=3)
    for name, arr in (("rp", rp.astype(np.int64)), ("col", col.astype(np.int32)), ("val", val.astype(np.float32)),
                      ("x", x), ("grp", G.row_ptr.astype(np.int64)), ("gcol", G.col.astype(np.int32))):
        arr.tofile(str(tmp_path / f"{name}.bin"))
    r = subprocess.run([exe, str(tmp_path), str(G.n), str(len(col)), str(len(G.col))], capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    y = np.fromfile(str(tmp_path / "y.bin"), np.float32)
    check(y, rp, col, val, x)
    k = int(r.stdout.strip())
    p = np.fromfile(str(tmp_path / "p.bin"), np.float32).astype(np.float64)
    ref, _ = oracle.pagerank(G.n, G.row_ptr, G.col, fixed_iters=k)
    assert np.abs(p - ref).sum() < 1e-6


def test_host_batch_edge_cases(gpu):
    """spmv_execute_host_batch: count 1, counts beyond the buffer depth, a rectangular matrix, the
    error paths (negative count, null pointers with count > 0); every product equals the device
    path bit for bit."""
    import ctypes
    import torch
    from paper_1103_2405_b200 import Plan, _capi
    rp, col, val = graphgen.random_csr(700, 1300, 20000, seed=9, kind="powerlaw", valued=True, signed=True)
    p = Plan(700, 1300, rp, col, val, device=0, tile_width=256, num_tiles=2, workload_size=128)
    for count in (1, 2, 7):
        X = np.stack([graphgen.uniform_f32(1300, seed=50 + b, mode=2) for b in range(count)])
        Y = p.execute_host_batch(X)
        assert Y.shape == (count, 700)
        for b in range(count):
            y = torch.empty(700, device="cuda")
            p.execute(torch.from_numpy(X[b]).cuda(), y)
            torch.cuda.synchronize()
            assert Y[b].tobytes() == y.cpu().numpy().tobytes()
            check(Y[b], rp, col, val, X[b])
    lib = _capi.lib()
    assert lib.spmv_execute_host_batch(p._h, None, None, -1, None) != 0
    assert lib.spmv_execute_host_batch(p._h, None, None, 3, None) != 0
    assert lib.spmv_execute_host_batch(p._h, None, None, 0, None) == 0


def test_plan_import_executes(gpu, tmp_path):
    """A plan written by spmv_plan_export and read back by spmv_plan_import (uploaded to the
    device) computes the bitwise-same product as the plan it came from."""
    import torch
    from paper_1103_2405_b200 import Plan
    rp, col, val = graphgen.random_csr(3000, 3000, 90000, seed=8, kind="powerlaw", valued=True)
    x = torch.from_numpy(graphgen.uniform_f32(3000, seed=3)).cuda()
    p = Plan(3000, 3000, rp, col, val, device=0, tile_width=256, num_tiles=3, workload_size=128)
    f = tmp_path / "plan.bin"
    p.export(f)
    q = Plan.load(f, device=0)
    y1, y2 = torch.empty(3000, device="cuda"), torch.empty(3000, device="cuda")
    p.execute(x, y1)
    q.execute(x, y2)
    torch.cuda.synchronize()
    assert y1.cpu().numpy().tobytes() == y2.cpu().numpy().tobytes()
    check(y2.cpu().numpy(), rp, col, val, x.cpu().numpy())
