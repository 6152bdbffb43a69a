"""CPU tests of the C-ABI library (no GPU): every symbol of include/spmv.h is exported, and the
product builder's layout is byte-identical to the independent numpy format oracle
(oracle/format_ref.py) on the same explicit parameters; layout -> COO equals the input."""
import ctypes
import json
import os
import re

import numpy as np
import pytest

import graphgen
from oracle import format_ref

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    from paper_1103_2405_b200 import _capi
    hdr = open(os.path.join(ROOT, "include", "spmv.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    names = set(re.findall(r"\b([a-z_][a-z0-9_]*)\s*\(", hdr))
    names -= {"if", "sizeof", "defined"}
    lib = ctypes.CDLL(_capi.LIB_PATH)
    missing = [n for n in sorted(names) if not hasattr(lib, n)]
    assert not missing, missing
    assert set(names) == set(_capi.SIGNATURES), set(names) ^ set(_capi.SIGNATURES)
    assert _capi.lib().spmv_version().startswith(b"tcspmv")


def build_both(nr, nc, rp, col, val, tw, T, wls, align=8, split=True, camping=False, ell_h=32, orient=0):
    from paper_1103_2405_b200 import Plan
    ref = format_ref.build(nr, nc, rp, col, val, tw, T, wls, align_rm=align, split_long_rows=split,
                           camping_pad=camping, ell_h=ell_h, orient=orient)
    p = Plan(nr, nc, rp, col, val, device=-1, tile_width=tw, num_tiles=T, workload_sizes=wls,
             align_rm=align, split_long_rows=int(split), camping_pad=int(camping), ell_h=ell_h,
             pattern=int(val is None), orient=orient)
    return ref, p


def assert_same(ref, p):
    L = p.layout()
    assert np.array_equal(L["perm"], ref.perm)
    assert np.array_equal(L["tiles"], ref.tiles)
    for k in ("off", "row_base", "w", "h", "kind", "kvec", "split_id", "chunk"):
        assert np.array_equal(L["desc"][k], ref.desc[k]), k
    assert np.array_equal(L["row_id"], ref.row_id)
    assert np.array_equal(L["slot_col"], ref.slot_col)
    if ref.slot_val is None:
        assert L["slot_val"] is None
    else:
        assert L["slot_val"].tobytes() == ref.slot_val.tobytes()
    assert np.array_equal(L["split"].reshape(-1, 3), ref.split.reshape(-1, 3))


def test_fig1_fixture_bit_exact():
    with open(os.path.join(ROOT, "tests", "golden", "fig1.json")) as f:
        g = json.load(f)
    ents = sorted(map(tuple, g["entries_row_col"]))
    rp = np.zeros(g["n_rows"] + 1, np.int64)
    for r, _ in ents:
        rp[r + 1] += 1
    rp = np.cumsum(rp)
    col = np.array([c for _, c in ents], np.int32)
    ref, p = build_both(8, 8, rp, col, None, 2, 2, [4, 4, 4], align=2, ell_h=2)
    assert_same(ref, p)


@pytest.mark.parametrize("seed", range(12))
def test_random_bit_exact(seed):
    rng = np.random.default_rng(1000 + seed)
    nr, nc = int(rng.integers(1, 600)), int(rng.integers(1, 600))
    kind = "powerlaw" if seed % 2 else "uniform"
    valued = seed % 3 != 0
    rp, col, val = graphgen.random_csr(nr, nc, int(rng.integers(0, 6000)), seed=seed, kind=kind,
                                       valued=valued, signed=bool(seed % 4 == 1))
    tw = int(rng.integers(1, 64))
    maxT = (nc + tw - 1) // tw
    T = int(rng.integers(0, min(maxT, 5) + 1))
    wls = [int(rng.integers(1, 300)) for _ in range(T + 1)]
    split = seed % 5 != 0
    if not split:
        # paper mode (reading R21): WL at least the longest row of every tile
        longest = int(np.diff(rp).max()) if nr else 1
        wls = [max(w, longest, 1) for w in wls]
    ref, p = build_both(nr, nc, rp, col, val, tw, T, wls, align=[4, 8, 32][seed % 3],
                        split=split, camping=seed % 4 == 2)
    assert_same(ref, p)
    r, c, v = p.to_coo()
    got = sorted(zip(r.tolist(), c.tolist(), v.tolist()))
    exp_v = np.ones(len(col), np.float32) if val is None else val
    exp = sorted(zip(np.repeat(np.arange(nr), np.diff(rp)).tolist(), col.tolist(), exp_v.tolist()))
    assert got == exp


@pytest.mark.parametrize("orient", [1, 2])
@pytest.mark.parametrize("seed", range(4))
def test_single_format_orientations_bit_exact(orient, seed):
    """f2 ablation layouts: row major only (CSR-vector) and column major only (ELL)."""
    rng = np.random.default_rng(2000 + seed)
    nr, nc = int(rng.integers(50, 500)), int(rng.integers(50, 500))
    rp, col, val = graphgen.random_csr(nr, nc, int(rng.integers(500, 6000)), seed=seed, kind="powerlaw",
                                       valued=seed % 2 == 0)
    tw = int(rng.integers(8, 64))
    T = int(rng.integers(0, 3))
    wls = [int(rng.integers(16, 300)) for _ in range(T + 1)]
    ref, p = build_both(nr, nc, rp, col, val, tw, T, wls, orient=orient)
    assert_same(ref, p)
    kind, w = ref.desc["kind"], ref.desc["w"]
    if orient == 1:      # only zero-length rows stay column major
        assert (w[kind == format_ref.KIND_CM] == 0).all()
    else:
        assert not (kind == format_ref.KIND_RM).any()
    r, c, v = p.to_coo()
    assert len(r) == len(col)


def test_graph_bit_exact_t_small():
    G = graphgen.make_graph("t_small")
    # PageRank's matrix is A^T (rows = targets)
    rpt, colt = graphgen.keys_to_csr(G.keys, G.n, transpose=True)
    ref, p = build_both(G.n, G.n, rpt, colt, None, 256, 3, [64, 128, 32, 512])
    assert_same(ref, p)


def test_paper_mode_rowsplit_error():
    from paper_1103_2405_b200 import Plan, SpmvError
    rp = np.array([0, 10, 11])
    col = np.concatenate([np.arange(10), [3]]).astype(np.int32)
    with pytest.raises(SpmvError, match="EROWSPLIT"):
        Plan(2, 10, rp, col, None, device=-1, tile_width=10, num_tiles=0, workload_sizes=[4],
             split_long_rows=0)
    Plan(2, 10, rp, col, None, device=-1, tile_width=10, num_tiles=0, workload_sizes=[10],
         split_long_rows=0)


@pytest.mark.parametrize("bad", ["rowptr", "col", "nrows"])
def test_invalid_inputs(bad):
    from paper_1103_2405_b200 import Plan, SpmvError
    rp = np.array([0, 2, 3]); col = np.array([0, 1, 1], np.int32)
    if bad == "rowptr":
        rp = np.array([0, 3, 2])
    if bad == "col":
        col = np.array([0, 5, 1], np.int32)
    with pytest.raises(SpmvError, match="EINVAL"):
        if bad == "nrows":
            Plan(-1, 2, rp, col, None, device=-1)
        else:
            Plan(2, 2, rp, col, None, device=-1)


def test_empty_matrix_and_zero_rows():
    from paper_1103_2405_b200 import Plan
    ref, p = build_both(5, 3, np.zeros(6, np.int64), np.zeros(0, np.int32), None, 2, 0, [16])
    assert_same(ref, p)
    L = p.layout()
    assert L["desc"]["w"].tolist() == [0] and L["desc"]["h"].tolist() == [32]
    rows = [int(e) & ((1 << 29) - 1) for e in L["row_id"] if e != 0xFFFFFFFF]
    assert rows == [0, 1, 2, 3, 4]


def test_no_device_means_loud_error():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has GPU")
    from paper_1103_2405_b200 import Plan, SpmvError
    with pytest.raises(SpmvError, match="ECUDA"):
        Plan(2, 2, np.array([0, 1, 2]), np.array([1, 0], np.int32), None, device=0)


def read_export(path):
    """Parse the spmv_plan_export file format (include/spmv.h) without the product's code."""
    b = open(path, "rb").read()
    assert b[:8] == b"TCSPMV1\0"
    hdr = np.frombuffer(b, np.int64, 8, 8)
    nr, nc, nw, ne, ns, nsp, nt, valued = (int(v) for v in hdr)
    pos = 72
    out = dict(n_rows=nr)

    def take(name, dt, count):
        nonlocal pos
        a = np.frombuffer(b, dt, count, pos)
        pos += a.nbytes
        out[name] = a

    take("perm", np.int32, nc)
    take("tiles", np.int64, 4 * nt)
    take("off", np.int64, nw)
    for k in ("row_base", "w", "h", "split_id", "chunk"):
        take(k, np.int32, nw)
    take("kind", np.uint8, nw)
    take("kvec", np.uint8, nw)
    take("row_id", np.uint32, ne)
    take("slot_col", np.int32, ns)
    if valued:
        take("slot_val", np.float32, ns)
    take("split", np.int32, 3 * nsp)
    assert pos == len(b)
    return out


@pytest.mark.parametrize("valued", [True, False])
def test_export_file_matches_format_oracle(tmp_path, valued):
    """spmv_plan_export writes the layout byte-identical to oracle/format_ref."""
    rp, col, val = graphgen.random_csr(300, 280, 4000, seed=5, kind="powerlaw")
    if not valued:
        val = None
    ref, p = build_both(300, 280, rp, col, val, 64, 2, [64, 128, 256])
    path = tmp_path / "plan.bin"
    p.export(path)
    E = read_export(path)
    assert np.array_equal(E["perm"], ref.perm)
    assert np.array_equal(E["tiles"].reshape(ref.tiles.shape), ref.tiles)
    for k in ("off", "row_base", "w", "h", "kind", "kvec", "split_id", "chunk"):
        assert np.array_equal(E[k], ref.desc[k]), k
    assert np.array_equal(E["row_id"], ref.row_id)
    assert np.array_equal(E["slot_col"], ref.slot_col)
    if valued:
        assert E["slot_val"].tobytes() == ref.slot_val.tobytes()
    else:
        assert "slot_val" not in E
    assert np.array_equal(E["split"].reshape(-1, 3), ref.split.reshape(-1, 3))


def test_plain_c_consumer(tmp_path):
    """The boundary is a C ABI: a C99 program compiled against include/spmv.h and linked to
    libtcspmv.so (no Python, no torch) partitions, builds a host-only plan and decodes it."""
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    libdir = os.path.join(root, "paper_1103_2405_b200", "lib")
    exe = str(tmp_path / "abi_consumer")
    r = subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(root, "include"),
                        os.path.join(root, "tests", "c", "abi_consumer.c"), "-L", libdir, "-ltcspmv",
                        "-Wl,-rpath," + libdir, "-o", exe], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and r.stdout.strip() == "ok", r.stdout + r.stderr


def test_parallel_transpose_equals_serial(tmp_path):
    """csrc/graph_build.h transpose (OpenMP, per-thread target ranges) is byte-equal to the serial
    counting scatter, hub rows included."""
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = str(tmp_path / "transpose_check")
    r = subprocess.run(["g++", "-O2", "-fopenmp", "-std=c++17", "-I", os.path.join(root, "paper_1103_2405_b200", "csrc"),
                        os.path.join(root, "tests", "c", "transpose_check.cpp"), "-o", exe], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.strip() == "ok", r.stdout + r.stderr


def test_keep_col_order_layout():
    """keep_col_order: the columns keep the caller's order (perm = identity, no dense tiles) and the
    layout still decodes to the input entries."""
    from paper_1103_2405_b200 import Plan
    rp, col, val = graphgen.random_csr(500, 700, 9000, seed=3, kind="powerlaw", valued=True)
    p = Plan(500, 700, rp, col, val, device=-1, keep_col_order=1)
    lay = p.layout()
    assert np.array_equal(lay["perm"], np.arange(700))
    assert p.stats()["num_tiles"] == 0
    r, c, v = p.to_coo()
    assert sorted(zip(r.tolist(), c.tolist(), v.tolist())) == sorted(
        zip(np.repeat(np.arange(500), np.diff(rp)).tolist(), col.tolist(), val.tolist()))


@pytest.mark.parametrize("seed", range(3))
def test_plan_import_roundtrip(seed, tmp_path):
    """spmv_plan_import reads back what spmv_plan_export wrote: re-exported byte for byte (every
    layout array), the same COO decode (host-only plans)."""
    from paper_1103_2405_b200 import Plan
    rng = np.random.default_rng(40 + seed)
    rp, col, val = graphgen.random_csr(400, 600, 8000, seed=seed, kind="powerlaw", valued=seed != 1)
    p = Plan(400, 600, rp, col, val, device=-1, tile_width=64, num_tiles=int(rng.integers(0, 4)),
             workload_size=int(rng.integers(16, 300)), two_phase=0)
    f = tmp_path / "plan.bin"
    p.export(f)
    q = Plan.load(f, device=-1)
    f2 = tmp_path / "plan2.bin"
    q.export(f2)
    assert f.read_bytes() == f2.read_bytes()
    assert q.stats()["nnz"] == len(col)
    r1, c1, v1 = p.to_coo()
    r2, c2, v2 = q.to_coo()
    assert sorted(zip(r1.tolist(), c1.tolist(), v1.tolist())) == sorted(zip(r2.tolist(), c2.tolist(), v2.tolist()))


def test_plan_import_rejects_garbage(tmp_path):
    from paper_1103_2405_b200 import Plan
    from paper_1103_2405_b200._capi import SpmvError
    f = tmp_path / "x.bin"
    f.write_bytes(b"not a plan at all")
    with pytest.raises(SpmvError):
        Plan.load(f, device=-1)


@pytest.mark.parametrize("seed", range(6))
def test_tile_coo_bit_exact(seed):
    """f2 TILE-COO (orient = 3): the dense tiles as COO workloads (whole rows back to back,
    row ends flagged), the remainder composite; byte-identical to the oracle builder and decoding
    to the input (split and paper mode both)."""
    rng = np.random.default_rng(3000 + seed)
    nr, nc = int(rng.integers(50, 700)), int(rng.integers(50, 700))
    valued = seed % 2 == 0
    rp, col, val = graphgen.random_csr(nr, nc, int(rng.integers(500, 9000)), seed=seed, kind="powerlaw",
                                       valued=valued)
    tw = int(rng.integers(4, 80))
    T = int(rng.integers(1, min((nc + tw - 1) // tw, 5) + 1))
    wls = [int(rng.integers(8, 400)) for _ in range(T + 1)]
    split = seed != 3
    if not split:
        longest = int(np.diff(rp).max())
        wls = [max(w, longest) for w in wls]
    ref, p = build_both(nr, nc, rp, col, val, tw, T, wls, split=split, orient=3)
    assert_same(ref, p)
    assert 3 in set(ref.desc["kind"].tolist())
    r, c, v = format_ref.decode_to_coo(ref)
    exp_v = np.ones(len(col)) if val is None else val
    assert sorted(zip(r.tolist(), c.tolist(), v.tolist())) == sorted(
        zip(np.repeat(np.arange(nr), np.diff(rp)).tolist(), col.tolist(), exp_v.astype(np.float64).tolist()))
    r2, c2, v2 = p.to_coo()
    assert sorted(zip(r2.tolist(), c2.tolist())) == sorted(zip(r.tolist(), c.tolist()))


def test_binding_rejects_bad_shapes():
    """The binding checks sizes before any C call (ValueError, also under python -O)."""
    from paper_1103_2405_b200 import Plan, Solver
    rp = np.array([0, 2, 3]); col = np.array([0, 1, 1], np.int32)
    with pytest.raises(ValueError):
        Plan(3, 2, rp, col, None, device=-1)               # len(row_ptr) != n_rows + 1
    with pytest.raises(ValueError):
        Plan(2, 2, rp, col[:2], None, device=-1)           # row_ptr[-1] > len(col)
    with pytest.raises(ValueError):
        Plan(2, 2, rp, col, np.ones(2, np.float32), device=-1)   # len(val) < nnz
    p = Plan(2, 2, rp, col, None, device=-1)
    with pytest.raises(ValueError):
        p.execute_host(np.ones(1, np.float32))             # x shorter than n_cols
    with pytest.raises(ValueError):
        p.execute_host_batch(np.ones((2, 3), np.float32))  # wrong X shape
    with pytest.raises(ValueError):
        Solver.local("rwr", 2, np.array([0, 1], np.int32), rp, col, out_degree=np.ones(3, np.int32))
