"""oracle -- TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct CPU reference for the tiled-composite SpMV path of Yang,
Parthasarathy & Sadayappan, "Fast Sparse Matrix-Vector Multiplication on GPUs: Implications for
Graph Mining", VLDB 2011.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / `--impl reference` legs may import this package.  It shares no code with the
product (paper_1103_2405_b200/): neither imports the other; only graphgen/ (inputs) serves both.

Parts (each cites the passage it follows; pins live in tests/test_oracle_*.py):
  spmv, pagerank, hits, rwr        fp64 C (oracle.c), plain definitions       -- pinned
  format_ref                       numpy layout builder (Solutions 1-3)        -- pinned
  partition_ref.bitonic_partition  snake order (Sec. 3.2)                      -- pinned
  model_ref                        Alg. 1-3 / Eq. 1-5 transcription            -- pinned
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def _lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make`")
        L = ctypes.CDLL(path)
        vp, i64, i32, d = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_double
        L.oracle_spmv.restype = None
        L.oracle_spmv.argtypes = [i64, vp, vp, vp, vp, vp, vp]
        L.oracle_pagerank.restype = ctypes.c_int
        L.oracle_pagerank.argtypes = [i64, vp, vp, d, d, i32, i32, vp, vp, vp]
        L.oracle_hits.restype = ctypes.c_int
        L.oracle_hits.argtypes = [i64, vp, vp, i32, d, i32, i32, vp, vp, vp, vp]
        L.oracle_rwr.restype = ctypes.c_int
        L.oracle_rwr.argtypes = [i64, vp, vp, i64, d, d, i32, i32, vp, vp, vp]
        _LIB = L
    return _LIB


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def spmv(row_ptr, col, val, x):
    """y = A x in fp64, plus b_i = sum |a_ij x_j| (tolerance scale).
    val None = pattern matrix (all ones).  x is fp32 (the product's input type)."""
    rp, cl, xx = _c(row_ptr, np.int64), _c(col, np.int32), _c(x, np.float32)
    n = len(rp) - 1
    vv = None if val is None else _c(val, np.float32)
    y = np.zeros(n, dtype=np.float64)
    b = np.zeros(n, dtype=np.float64)
    _lib().oracle_spmv(n, rp.ctypes.data, cl.ctypes.data if len(cl) else None,
                       None if vv is None else (vv.ctypes.data if len(vv) else None),
                       xx.ctypes.data if len(xx) else None, y.ctypes.data if n else None,
                       b.ctypes.data if n else None)
    return y, b


class IterResult:
    def __init__(self, iterations, residual, converged):
        self.iterations, self.residual, self.converged = iterations, residual, converged


def pagerank(n, row_ptr, col, c=0.85, tol=1e-6, max_iter=1000, fixed_iters=0):
    """Eq. 6 with uniform redistribution of dangling mass (R1).
    Adjacency CSR: row u lists targets v of u->v.  Returns (p fp64, IterResult)."""
    rp, cl = _c(row_ptr, np.int64), _c(col, np.int32)
    p = np.zeros(n, dtype=np.float64)
    it, res = ctypes.c_int32(0), ctypes.c_double(0)
    rc = _lib().oracle_pagerank(n, rp.ctypes.data, cl.ctypes.data if len(cl) else None, c, tol,
                                max_iter, fixed_iters, p.ctypes.data, ctypes.byref(it), ctypes.byref(res))
    return p, IterResult(it.value, res.value, rc == 0)


def hits(n, row_ptr, col, norm=2, tol=1e-6, max_iter=1000, fixed_iters=0):
    """Eq. 7-8, Jacobi update, halves normalised (L2 default; 1 = sum 1)."""
    rp, cl = _c(row_ptr, np.int64), _c(col, np.int32)
    a = np.zeros(n, dtype=np.float64)
    h = np.zeros(n, dtype=np.float64)
    it, res = ctypes.c_int32(0), ctypes.c_double(0)
    rc = _lib().oracle_hits(n, rp.ctypes.data, cl.ctypes.data if len(cl) else None, norm, tol,
                            max_iter, fixed_iters, a.ctypes.data, h.ctypes.data,
                            ctypes.byref(it), ctypes.byref(res))
    return a, h, IterResult(it.value, res.value, rc == 0)


def rwr(n, row_ptr, col, query, c=0.9, tol=1e-6, max_iter=1000, fixed_iters=0):
    """Eq. 9 on binary(A u A^T), W column-normalised, r(0) = e_q."""
    rp, cl = _c(row_ptr, np.int64), _c(col, np.int32)
    r = np.zeros(n, dtype=np.float64)
    it, res = ctypes.c_int32(0), ctypes.c_double(0)
    rc = _lib().oracle_rwr(n, rp.ctypes.data, cl.ctypes.data if len(cl) else None, query, c, tol,
                           max_iter, fixed_iters, r.ctypes.data, ctypes.byref(it), ctypes.byref(res))
    return r, IterResult(it.value, res.value, rc == 0)
