"""graphgen -- seeded synthetic inputs, shared by the oracle and the product path.

Holds none of the method's arithmetic: it only draws graphs and vectors (counter-based
splitmix64, so every consumer sees the same bits).  Input recipe: DESIGN.md "Inputs".

Stand-ins for the paper's datasets (Table 2, L307-L313 Table 3), which are
not shipped.  The named configs follow BASELINE.json "configs" as made concrete in SURVEY.md 8(d).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

# seeds (SURVEY.md 8(d) "Generator protocol")
SEED_GRAPH, SEED_RELABEL, SEED_X, SEED_VAL, SEED_QUERY = 1, 2, 3, 4, 5


def _lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "libgraphgen.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make` (or __graft_entry__.build())")
        L = ctypes.CDLL(path)
        u64p = ctypes.POINTER(ctypes.c_uint64)
        L.gg_draw.restype = ctypes.c_uint64
        L.gg_draw.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        L.gg_rmat.restype = ctypes.c_int
        L.gg_rmat.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_double,
                              ctypes.c_double, ctypes.c_double, ctypes.c_uint64, ctypes.c_uint64,
                              ctypes.POINTER(u64p), ctypes.POINTER(ctypes.c_int64)]
        L.gg_chung_lu.restype = ctypes.c_int
        L.gg_chung_lu.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_double, ctypes.c_double,
                                  ctypes.c_uint64, ctypes.c_uint64, ctypes.POINTER(u64p),
                                  ctypes.POINTER(ctypes.c_int64)]
        L.gg_keys_to_csr.restype = None
        L.gg_keys_to_csr.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
                                     ctypes.c_void_p, ctypes.c_void_p]
        L.gg_uniform_f32.restype = None
        L.gg_uniform_f32.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int64, ctypes.c_int,
                                     ctypes.c_void_p]
        L.gg_edge_values_f32.restype = None
        L.gg_edge_values_f32.argtypes = [ctypes.c_uint64, ctypes.c_void_p, ctypes.c_int64,
                                         ctypes.c_int, ctypes.c_void_p]
        L.gg_free.restype = None
        L.gg_free.argtypes = [ctypes.c_void_p]
        _LIB = L
    return _LIB


def _take_keys(ptr, m) -> np.ndarray:
    L = _lib()
    if m.value == 0:
        L.gg_free(ctypes.cast(ptr, ctypes.c_void_p))
        return np.zeros(0, dtype=np.uint64)
    arr = np.ctypeslib.as_array(ptr, shape=(m.value,)).copy()
    L.gg_free(ctypes.cast(ptr, ctypes.c_void_p))
    return arr


def rmat_edges(scale: int, n: int, m: int, a=0.57, b=0.19, c=0.19, seed=SEED_GRAPH,
               relabel_seed=SEED_RELABEL) -> np.ndarray:
    """m unique directed edges (no self loops) of an R-MAT graph on a 2^scale grid, ids >= n
    rejected, then a seeded random relabel.  Returns sorted keys (u << 32) | v."""
    ptr = ctypes.POINTER(ctypes.c_uint64)()
    mo = ctypes.c_int64(0)
    rc = _lib().gg_rmat(scale, n, m, a, b, c, seed, relabel_seed, ctypes.byref(ptr), ctypes.byref(mo))
    if rc != 0:
        raise ValueError(f"gg_rmat failed rc={rc}")
    return _take_keys(ptr, mo)


def chung_lu_edges(n: int, m: int, alpha: float, max_deg: float = 2e4, seed=SEED_GRAPH,
                   relabel_seed=SEED_RELABEL) -> np.ndarray:
    """m unique directed edges of a capped Chung-Lu graph, weight_i = (i+i0)^(-1/(alpha-1))."""
    ptr = ctypes.POINTER(ctypes.c_uint64)()
    mo = ctypes.c_int64(0)
    rc = _lib().gg_chung_lu(n, m, alpha, max_deg, seed, relabel_seed, ctypes.byref(ptr), ctypes.byref(mo))
    if rc != 0:
        raise ValueError(f"gg_chung_lu failed rc={rc}")
    return _take_keys(ptr, mo)


def keys_to_csr(keys: np.ndarray, n: int, transpose: bool = False):
    """Sorted unique edge keys -> CSR (row_ptr int64 [n+1], col int32 [m]).
    transpose=False: row u lists targets v (adjacency A);  True: row v lists sources u (A^T)."""
    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    rp = np.zeros(n + 1, dtype=np.int64)
    col = np.zeros(max(len(keys), 1), dtype=np.int32)
    _lib().gg_keys_to_csr(keys.ctypes.data, len(keys), n, int(transpose), rp.ctypes.data, col.ctypes.data)
    return rp, col[: len(keys)]


def uniform_f32(count: int, seed=SEED_X, mode: int = 0, offset: int = 0) -> np.ndarray:
    """mode 0: U[0,1); 1: U(0,1]; 2: U(-1,1) without 0.  24-bit exact fp32."""
    out = np.empty(max(count, 1), dtype=np.float32)
    _lib().gg_uniform_f32(seed, offset, count, mode, out.ctypes.data)
    return out[:count]


def edge_values(keys: np.ndarray, seed=SEED_VAL, mode: int = 1) -> np.ndarray:
    """per-edge fp32 values keyed by the edge key (storage-order independent)."""
    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    out = np.empty(max(len(keys), 1), dtype=np.float32)
    _lib().gg_edge_values_f32(seed, keys.ctypes.data, len(keys), mode, out.ctypes.data)
    return out[: len(keys)]


def draw(seed: int, k: int) -> int:
    return int(_lib().gg_draw(seed, k))


@dataclass
class Graph:
    """A directed graph: n vertices, sorted unique edge keys, adjacency CSR (row u -> targets)."""
    name: str
    n: int
    keys: np.ndarray
    row_ptr: np.ndarray
    col: np.ndarray

    @property
    def m(self) -> int:
        return int(len(self.keys))


def graph_from_keys(name: str, n: int, keys: np.ndarray) -> Graph:
    rp, col = keys_to_csr(keys, n, transpose=False)
    return Graph(name, n, keys, rp, col)


# Named workloads (BASELINE.json configs).
CONFIGS = {
    # c1: R-MAT scale 16, edge factor 16, Graph500 (a,b,c) = (.57,.19,.19)
    "c1": dict(kind="rmat", scale=16, n=65536, m=1_000_000, a=0.57, b=0.19, c=0.19),
    # c2: LiveJournal-shaped (soc-LiveJournal1 sizes), R-MAT (a,b,c,d) = (.50,.20,.20,.10)
    "c2": dict(kind="rmat", scale=23, n=4_847_571, m=68_993_773, a=0.50, b=0.20, c=0.20),
    # c3: Flickr / YouTube shaped capped Chung-Lu skew sweep (alpha in 1.8..2.6)
    "c3_flickr": dict(kind="chung_lu", n=1_700_000, m=22_600_000, alpha=2.2, max_deg=2e4),
    "c3_youtube": dict(kind="chung_lu", n=1_100_000, m=4_900_000, alpha=2.2, max_deg=2e4),
    # c4: it-2004 shaped web graph, Graph500 R-MAT scale 26, ids >= n rejected
    "c4": dict(kind="rmat", scale=26, n=41_291_594, m=1_150_725_436, a=0.57, b=0.19, c=0.19),
    # c5: uk-union shaped web graph, Graph500 R-MAT scale 28, ids >= n rejected (HITS
    # block 267,266,080 rows, 11,015,359,644 entries).  Device generator only (DeviceGraph): the host
    # generator would need ~200 GB.  c5_s22: the same shape at 1/64 (dry runs of the c5 route).
    "c5": dict(kind="rmat", scale=28, n=133_633_040, m=5_507_679_822, a=0.57, b=0.19, c=0.19),
    "c5_s22": dict(kind="rmat", scale=22, n=2_088_016, m=86_057_497, a=0.57, b=0.19, c=0.19),
    # small parity cases (several tiles + ragged tails, oracle finishes in seconds)
    "t_small": dict(kind="rmat", scale=12, n=4000, m=40_000, a=0.57, b=0.19, c=0.19),
    "t_mid": dict(kind="rmat", scale=17, n=100_000, m=1_200_000, a=0.50, b=0.20, c=0.20),
}


def make_graph(config: str, **override) -> Graph:
    spec = dict(CONFIGS[config])
    spec.update(override)
    kind = spec.pop("kind")
    if kind == "rmat":
        keys = rmat_edges(spec["scale"], spec["n"], spec["m"], spec["a"], spec["b"], spec["c"],
                          spec.get("seed", SEED_GRAPH), spec.get("relabel_seed", SEED_RELABEL))
    else:
        keys = chung_lu_edges(spec["n"], spec["m"], spec["alpha"], spec.get("max_deg", 2e4),
                              spec.get("seed", SEED_GRAPH), spec.get("relabel_seed", SEED_RELABEL))
    return graph_from_keys(config, spec["n"], keys)


def dense_csr(n_rows: int, n_cols: int, seed: int = SEED_VAL):
    """Appendix D's dense case: every entry stored, values U(0,1] from the counter
    generator.  Returns (row_ptr, col, val)."""
    rp = np.arange(n_rows + 1, dtype=np.int64) * n_cols
    col = np.tile(np.arange(n_cols, dtype=np.int32), n_rows)
    val = uniform_f32(n_rows * n_cols, seed=seed, mode=1)
    return rp, col, val


def banded_csr(n: int, half_band: int, seed: int = SEED_VAL, drop: float = 0.0):
    """Unstructured-mesh-like banded matrix (Appendix D, FEM-like): row i holds the columns
    [i - half_band, i + half_band] clipped to [0, n); with drop > 0 each off-diagonal entry is
    removed with that probability (a ragged band).  Values U(0,1].  Returns (row_ptr, col, val)."""
    rng = np.random.default_rng(seed)
    off = np.arange(-half_band, half_band + 1)
    r = np.repeat(np.arange(n, dtype=np.int64), len(off))
    c = r + np.tile(off, n)
    keep = (c >= 0) & (c < n)
    if drop > 0:
        keep &= (c == r) | (rng.random(len(c)) >= drop)
    r, c = r[keep], c[keep]
    rp = np.zeros(n + 1, dtype=np.int64)
    np.add.at(rp, r + 1, 1)
    rp = np.cumsum(rp)
    val = uniform_f32(len(c), seed=seed, mode=1)
    return rp, c.astype(np.int32), val


def random_csr(n_rows: int, n_cols: int, nnz: int, seed: int = 7, kind: str = "uniform",
               valued: bool = True, signed: bool = False, alpha: float = 2.0):
    """Small random sparse matrices for parity/format tests (rectangular allowed, duplicates
    allowed so the 'entries kept as given' rule is exercised).  kind = 'uniform' or 'powerlaw'
    (column and row ids drawn from a Zipf-like weight).  Returns (row_ptr, col, val|None)."""
    rng = np.random.default_rng(seed)
    if kind == "uniform":
        r = rng.integers(0, max(n_rows, 1), size=nnz)
        c = rng.integers(0, max(n_cols, 1), size=nnz)
    else:
        def zipf_ids(n, size):
            w = (np.arange(n) + 1.0) ** (-1.0 / (alpha - 1.0))
            w /= w.sum()
            ids = rng.choice(n, size=size, p=w)
            return rng.permutation(n)[ids]
        r = zipf_ids(n_rows, nnz)
        c = zipf_ids(n_cols, nnz)
    order = np.lexsort((c, r))
    r, c = r[order], c[order]
    rp = np.zeros(n_rows + 1, dtype=np.int64)
    np.add.at(rp, r + 1, 1)
    rp = np.cumsum(rp).astype(np.int64)
    col = c.astype(np.int32)
    val = None
    if valued:
        val = (rng.uniform(-1, 1, nnz) if signed else rng.uniform(0, 1, nnz) + 1e-3).astype(np.float32)
    return rp, col, val


# ---------------------------------------------------------------- the same generator on the device
# (graphgen_gpu.cu: c4 / c5 sizes, and one rank's rows without the whole edge list on the host)
_GLIB = None


def _glib():
    global _GLIB
    if _GLIB is None:
        path = os.path.join(_HERE, "libgraphgen_gpu.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make` (or __graft_entry__.build())")
        L = ctypes.CDLL(path)
        u64p = ctypes.POINTER(ctypes.c_uint64)
        i32p = ctypes.POINTER(ctypes.c_int32)
        L.ggg_last_error.restype = ctypes.c_char_p
        L.ggg_rmat.restype = ctypes.c_int
        L.ggg_rmat.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_double, ctypes.c_double,
                               ctypes.c_double, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int,
                               ctypes.POINTER(u64p), ctypes.POINTER(ctypes.c_int64)]
        L.ggg_free.argtypes = [ctypes.c_void_p]
        L.ggg_free.restype = None
        L.ggg_host_free.argtypes = [ctypes.c_void_p]
        L.ggg_host_free.restype = None
        L.ggg_to_host.restype = ctypes.c_int
        L.ggg_to_host.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]
        L.ggg_degrees.restype = ctypes.c_int
        L.ggg_degrees.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
        L.ggg_owned_cols.restype = ctypes.c_int
        L.ggg_owned_cols.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p,
                                     ctypes.c_int32, ctypes.POINTER(i32p), ctypes.POINTER(ctypes.c_int64)]
        _GLIB = L
    return _GLIB


def _gcheck(rc, what):
    if rc != 0:
        raise RuntimeError(f"{what} failed rc={rc}: {_glib().ggg_last_error().decode()}")


# iteration-matrix kinds of DeviceGraph.owned_rows
KIND_A, KIND_AT, KIND_HITS = 0, 1, 2


class DeviceGraph:
    """The keys of make_graph(config) (R-MAT configs only), generated on `device` and kept there.
    Bit-identical to the host generator.  Free with close() (the keys of c5 take 44 GB)."""

    def __init__(self, config: str, device: int = 0, **override):
        spec = dict(CONFIGS[config])
        spec.update(override)
        if spec.pop("kind") != "rmat":
            raise ValueError("DeviceGraph: R-MAT configurations only")
        self.name, self.n, self.device = config, int(spec["n"]), device
        ptr = ctypes.POINTER(ctypes.c_uint64)()
        mo = ctypes.c_int64(0)
        _gcheck(_glib().ggg_rmat(spec["scale"], spec["n"], spec["m"], spec["a"], spec["b"], spec["c"],
                                 spec.get("seed", SEED_GRAPH), spec.get("relabel_seed", SEED_RELABEL), device,
                                 ctypes.byref(ptr), ctypes.byref(mo)), "ggg_rmat")
        self._d = ctypes.cast(ptr, ctypes.c_void_p).value
        self.m = int(mo.value)
        self._deg = None

    def close(self):
        if self._d:
            _glib().ggg_free(ctypes.c_void_p(self._d))
            self._d = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def keys(self) -> np.ndarray:
        out = np.empty(max(self.m, 1), dtype=np.uint64)
        _gcheck(_glib().ggg_to_host(ctypes.c_void_p(self._d), self.m, out.ctypes.data), "ggg_to_host")
        return out[: self.m]

    def degrees(self):
        """(out_degree, in_degree), int32 [n] each."""
        if self._deg is None:
            od = np.empty(self.n, dtype=np.int32)
            idg = np.empty(self.n, dtype=np.int32)
            _gcheck(_glib().ggg_degrees(ctypes.c_void_p(self._d), self.m, self.n, od.ctypes.data, idg.ctypes.data),
                    "ggg_degrees")
            self._deg = (od, idg)
        return self._deg

    def row_lengths(self, kind: int) -> np.ndarray:
        """Row lengths of the iteration matrix (int64): A (out-degree), A^T (in-degree) or the HITS
        block [[0, A^T], [A, 0]] (in-degrees then out-degrees)."""
        od, idg = self.degrees()
        if kind == KIND_A:
            return od.astype(np.int64)
        if kind == KIND_AT:
            return idg.astype(np.int64)
        return np.concatenate([idg, od]).astype(np.int64)

    def owned_rows(self, kind: int, owner: np.ndarray, q: int):
        """Rank q's rows of the iteration matrix: (owned_ids int32 ascending, row_ptr int64, col int32),
        columns ascending within each row (global ids; HITS block: rows v < n hold n + u)."""
        owner = np.ascontiguousarray(owner, dtype=np.int32)
        lens = self.row_lengths(kind)
        if len(owner) != len(lens):
            raise ValueError("owner must cover every row of the iteration matrix")
        ids = np.nonzero(owner == q)[0]
        rp = np.zeros(len(ids) + 1, dtype=np.int64)
        np.cumsum(lens[ids], out=rp[1:])
        ptr = ctypes.POINTER(ctypes.c_int32)()
        cnt = ctypes.c_int64(0)
        _gcheck(_glib().ggg_owned_cols(ctypes.c_void_p(self._d), self.m, self.n, kind, owner.ctypes.data, q,
                                       ctypes.byref(ptr), ctypes.byref(cnt)), "ggg_owned_cols")
        c = int(cnt.value)
        if c != int(rp[-1]):
            _glib().ggg_host_free(ctypes.cast(ptr, ctypes.c_void_p))
            raise RuntimeError(f"owned_rows: {c} columns for row lengths summing to {int(rp[-1])}")
        col = np.ctypeslib.as_array(ptr, shape=(max(c, 1),))[:c].copy()
        _glib().ggg_host_free(ctypes.cast(ptr, ctypes.c_void_p))
        return ids.astype(np.int32), rp, col
