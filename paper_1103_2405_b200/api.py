"""Thin Python binding over libtcspmv.so (include/spmv.h): argument marshalling only.

PyTorch is used for device memory and streams (tensors' data_ptr / current stream); every step
of the SpMV and of the power iterations runs in the library's CUDA kernels.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _capi as C
from ._capi import check

ALGO = {"pagerank": 0, "hits": 1, "rwr": 2}


def _np(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def _ptr(a):
    return None if a is None or a.size == 0 else a.ctypes.data


def _need(cond, msg):
    """argument validation that survives `python -O` (the C side trusts sizes it is given)"""
    if not cond:
        raise ValueError(msg)


def _csr(n_rows, row_ptr, col, what="matrix"):
    rp = _np(row_ptr, np.int64)
    cl = _np(col, np.int32)
    if int(n_rows) < 0:          # the library reports it (SPMV_EINVAL)
        return rp, cl
    _need(rp.ndim == 1 and len(rp) == int(n_rows) + 1, f"{what}: len(row_ptr) must be n_rows + 1 = {int(n_rows) + 1}")
    _need(len(rp) == 0 or (rp[0] == 0 and int(rp[-1]) <= len(cl)), f"{what}: row_ptr[0] must be 0 and row_ptr[-1] <= len(col)")
    return rp, cl


def _dev_vec(t, n, name):
    _need(hasattr(t, "data_ptr") and getattr(t, "is_cuda", False), f"{name} must be a CUDA tensor")
    _need(str(t.dtype) == "torch.float32", f"{name} must be float32")
    _need(t.is_contiguous(), f"{name} must be contiguous")
    _need(t.numel() >= n, f"{name} has {t.numel()} elements, needs {n}")


def make_options(**kw) -> C.Options:
    """spmv_options with defaults (spmv_options_default) overridden by keyword arguments.
    workload_sizes may be a list (num_tiles + 1 values)."""
    o = C.Options()
    C.lib().spmv_options_default(ctypes.byref(o))
    keep = {}
    for k, v in kw.items():
        if v is None:
            continue
        if k == "workload_sizes":
            arr = (ctypes.c_int32 * len(v))(*[int(x) for x in v])
            keep["wls"] = arr
            o.workload_sizes = ctypes.cast(arr, ctypes.POINTER(ctypes.c_int32))
        elif k == "perf_table_path":
            b = str(v).encode()
            keep["ptp"] = b
            o.perf_table_path = b
        else:
            if not hasattr(o, k):
                raise TypeError(f"unknown option {k}")
            setattr(o, k, int(v))
    o._keep = keep
    return o


def _stream_handle(stream):
    if stream is None:
        try:
            import torch
            if torch.cuda.is_available():
                return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        except Exception:
            pass
        return None
    if isinstance(stream, int):
        return ctypes.c_void_p(stream)
    return ctypes.c_void_p(stream.cuda_stream)


def _stats_dict(s: C.PlanStats) -> dict:
    T = s.num_tiles + 1
    return dict(n_rows=s.n_rows, n_cols=s.n_cols, nnz=s.nnz, num_tiles=s.num_tiles,
                tile_width=s.tile_width, n_workloads=s.n_workloads, n_slots=s.n_slots,
                n_row_entries=s.n_row_entries, n_split=s.n_split, n_chunks=s.n_chunks,
                device_bytes=s.device_bytes, predicted_us=s.predicted_us, build_ms=s.build_ms,
                wl=list(s.wl[:T]), tile_nnz=list(s.tile_nnz[:T]), tile_rows=list(s.tile_rows[:T]),
                tile_col_lo=list(s.tile_col_lo[:T]), tile_col_hi=list(s.tile_col_hi[:T]),
                tile_staged=list(s.tile_staged[:T]),
                tile_predicted_us=list(s.tile_predicted_us[:T]),
                composite_threshold=list(s.composite_threshold[:T]),
                resident_warps=s.resident_warps, perf_table_loaded=bool(s.perf_table_loaded),
                two_phase=bool(s.two_phase), pb_groups=s.pb_groups, pb_chunks=s.pb_chunks,
                pb_bins=s.pb_bins, pb_long_bins=s.pb_long_bins,
                one_pass_predicted_us=s.one_pass_predicted_us,
                two_phase_predicted_us=s.two_phase_predicted_us, orient=s.orient)


class Plan:
    """Tiled-composite plan of a sparse matrix (spmv_plan_create).  device=-1: host-only plan."""

    def __init__(self, n_rows, n_cols, row_ptr, col, val=None, device=0, **options):
        self.n_rows, self.n_cols = int(n_rows), int(n_cols)
        rp, cl = _csr(self.n_rows, row_ptr, col, "Plan")
        vv = None if val is None else _np(val, np.float32)
        _need(vv is None or len(vv) >= int(rp[-1]), "Plan: len(val) < nnz")
        if vv is None:
            options.setdefault("pattern", 1)
        self.nnz = int(rp[-1]) if len(rp) else 0
        self._opt = make_options(**options)
        h = ctypes.c_void_p()
        st = C.lib().spmv_plan_create(self.n_rows, self.n_cols, self.nnz, rp.ctypes.data, _ptr(cl),
                                      _ptr(vv), ctypes.byref(self._opt), int(device), ctypes.byref(h))
        check(st, "spmv_plan_create")
        self._h = h
        self.device = device

    def close(self):
        if getattr(self, "_h", None):
            C.lib().spmv_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- execution (device tensors) ------------------------------------------------------
    def execute(self, x, y, stream=None, permuted=False):
        """y = A x on device tensors (float32, contiguous); asynchronous on `stream`."""
        _dev_vec(x, self.n_cols, "x")
        _dev_vec(y, self.n_rows, "y")
        fn = C.lib().spmv_execute_permuted if permuted else C.lib().spmv_execute
        check(fn(self._h, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr()),
                 _stream_handle(stream)), "spmv_execute")
        return y

    def execute_host(self, x: np.ndarray, stream=None) -> np.ndarray:
        """host x -> device -> host y (copies inside; synchronises)."""
        xh = _np(x, np.float32)
        _need(xh.ndim == 1 and len(xh) >= self.n_cols, f"x needs {self.n_cols} elements")
        y = np.empty(max(self.n_rows, 1), dtype=np.float32)
        check(C.lib().spmv_execute_host(self._h, _ptr(xh) or ctypes.c_void_p(0), y.ctypes.data,
                                        _stream_handle(stream)), "spmv_execute_host")
        return y[: self.n_rows]

    def execute_host_batch(self, X, Y=None, stream=None):
        """Y[b] = A X[b] for host arrays X [count, n_cols] -> Y [count, n_rows] (numpy or pinned
        torch CPU tensors); copies in and out overlap the products (spmv_execute_host_batch)."""
        if Y is None:
            Y = np.empty((X.shape[0], self.n_rows), dtype=np.float32)
        count = int(X.shape[0])
        _need(tuple(Y.shape) == (count, self.n_rows) and tuple(X.shape) == (count, self.n_cols),
              f"X must be [count, {self.n_cols}] and Y [count, {self.n_rows}]")
        for t, nm in ((X, "X"), (Y, "Y")):
            if hasattr(t, "data_ptr"):
                _need(not t.is_cuda, f"{nm} must be a host (ideally pinned) tensor")
                _need(str(t.dtype) == "torch.float32" and t.is_contiguous(), f"{nm} must be contiguous float32")
            else:
                _need(t.flags.c_contiguous and t.dtype == np.float32, f"{nm} must be contiguous float32")
        xp = X.data_ptr() if hasattr(X, "data_ptr") else X.ctypes.data
        yp = Y.data_ptr() if hasattr(Y, "data_ptr") else Y.ctypes.data
        check(C.lib().spmv_execute_host_batch(self._h, ctypes.c_void_p(xp), ctypes.c_void_p(yp), count,
                                              _stream_handle(stream)), "spmv_execute_host_batch")
        return Y

    @property
    def launches(self) -> int:
        return int(C.lib().spmv_plan_launches(self._h))

    def stats(self) -> dict:
        s = C.PlanStats()
        check(C.lib().spmv_plan_stats(self._h, ctypes.byref(s)), "spmv_plan_stats")
        return _stats_dict(s)

    def layout(self) -> dict:
        """Copies of the layout arrays (Format v1) for byte-for-byte comparison."""
        v = C.LayoutView()
        check(C.lib().spmv_plan_layout(self._h, ctypes.byref(v)), "spmv_plan_layout")

        def arr(p, n, dt):
            if n == 0 or not p:
                return np.zeros(0, dtype=dt)
            return np.ctypeslib.as_array(p, shape=(n,)).astype(dt, copy=True)
        nw, nr, ns = v.n_workloads, v.n_row_entries, v.n_slots
        return dict(
            perm=arr(v.perm, v.n_cols, np.int32),
            tiles=arr(v.tiles, 4 * v.n_tiles_total, np.int64).reshape(-1, 4),
            desc=dict(off=arr(v.desc_off, nw, np.int64), row_base=arr(v.desc_row_base, nw, np.int32),
                      w=arr(v.desc_w, nw, np.int32), h=arr(v.desc_h, nw, np.int32),
                      kind=arr(v.desc_kind, nw, np.uint8), kvec=arr(v.desc_kvec, nw, np.uint8),
                      split_id=arr(v.desc_split_id, nw, np.int32), chunk=arr(v.desc_chunk, nw, np.int32)),
            row_id=arr(v.row_id, nr, np.uint32),
            slot_col=arr(v.slot_col, ns, np.int32),
            slot_val=None if not v.slot_val else arr(v.slot_val, ns, np.float32),
            split=arr(v.split, 3 * v.n_split, np.int32).reshape(-1, 3),
        )

    def export(self, path: str) -> None:
        """spmv_plan_export: the layout arrays as one binary file (include/spmv.h)."""
        check(C.lib().spmv_plan_export(self._h, str(path).encode()), "spmv_plan_export")

    @classmethod
    def load(cls, path: str, device=0):
        """spmv_plan_import: a plan from a file written by export() (preprocessing checkpoint)."""
        self = cls.__new__(cls)
        h = ctypes.c_void_p()
        check(C.lib().spmv_plan_import(str(path).encode(), int(device), ctypes.byref(h)), "spmv_plan_import")
        self._h = h
        self.device = device
        s = self.stats()
        self.n_rows, self.n_cols, self.nnz = s["n_rows"], s["n_cols"], s["nnz"]
        return self

    def to_coo(self):
        r = np.zeros(max(self.nnz, 1), np.int32)
        c = np.zeros(max(self.nnz, 1), np.int32)
        v = np.zeros(max(self.nnz, 1), np.float32)
        check(C.lib().spmv_plan_to_coo(self._h, r.ctypes.data, c.ctypes.data, v.ctypes.data),
              "spmv_plan_to_coo")
        return r[: self.nnz], c[: self.nnz], v[: self.nnz]


def iter_opts(algo: str, **kw) -> C.IterOpts:
    o = C.IterOpts()
    C.lib().spmv_iter_opts_default(ctypes.byref(o), ALGO[algo])
    for k, v in kw.items():
        if v is not None:
            setattr(o, k, v)
    return o


class Solver:
    """A power-iteration solver (PageRank / HITS / RWR) with its plan built once (L98)."""

    def __init__(self, algo: str, n, row_ptr, col, device=0, comm=None, iter_kw=None, **options):
        self.algo, self.n = algo, int(n)
        self._comm = comm                      # the communicator must outlive the solver
        rp, cl = _csr(self.n, row_ptr, col, "Solver")
        self.m = int(rp[-1])
        self._it = iter_opts(algo, **(iter_kw or {}))
        self._opt = make_options(**options)
        h = ctypes.c_void_p()
        check(C.lib().spmv_solver_create(ALGO[algo], self.n, self.m, rp.ctypes.data, _ptr(cl),
                                         ctypes.byref(self._it), ctypes.byref(self._opt),
                                         comm._h if comm is not None else None, int(device),
                                         ctypes.byref(h)), "spmv_solver_create")
        self._h = h

    @classmethod
    def local(cls, algo: str, n_global, owned_ids, row_ptr, col, out_degree=None, device=0, comm=None,
              iter_kw=None, **options):
        """Row-partitioned solver from this rank's rows only (spmv_solver_create_local)."""
        self = cls.__new__(cls)
        self.algo, self.n = algo, int(n_global)
        self._comm = comm
        ids = _np(owned_ids, np.int32)
        rp, cl = _csr(len(ids), row_ptr, col, "Solver.local")
        deg = _np(out_degree, np.int32) if out_degree is not None else None
        _need(deg is None or len(deg) == len(ids), "Solver.local: len(out_degree) must equal len(owned_ids)")
        self.m = int(rp[-1]) if len(rp) else 0
        self._it = iter_opts(algo, **(iter_kw or {}))
        self._opt = make_options(**options)
        h = ctypes.c_void_p()
        check(C.lib().spmv_solver_create_local(ALGO[algo], self.n, len(ids), _ptr(ids), rp.ctypes.data, _ptr(cl),
                                               _ptr(deg) if deg is not None else None, ctypes.byref(self._it),
                                               ctypes.byref(self._opt), comm._h if comm is not None else None,
                                               int(device), ctypes.byref(h)), "spmv_solver_create_local")
        self._h = h
        return self

    def run(self, query: int = 0, stream=None) -> dict:
        r = C.IterResult()
        st = C.lib().spmv_solver_run(self._h, int(query), _stream_handle(stream), ctypes.byref(r))
        if st not in (0, 10):
            check(st, "spmv_solver_run")
        return dict(iterations=r.iterations, converged=bool(r.converged), residual=r.residual,
                    ms_total=r.ms_total, us_per_iter=r.us_per_iter,
                    predicted_us_per_iter=r.predicted_us_per_iter, phase_us=list(r.phase_us))

    def run_batch(self, queries, stream=None) -> dict:
        """Batched RWR: all queries (<= 32) iterate together (spmv_solver_run_batch)."""
        q = _np(queries, np.int64)
        self._nq = len(q)
        r = C.IterResult()
        st = C.lib().spmv_solver_run_batch(self._h, q.ctypes.data, len(q), _stream_handle(stream), ctypes.byref(r))
        if st not in (0, 10):
            check(st, "spmv_solver_run_batch")
        return dict(iterations=r.iterations, converged=bool(r.converged), residual=r.residual,
                    ms_total=r.ms_total, us_per_iter=r.us_per_iter)

    def result_batch(self) -> np.ndarray:
        out = np.zeros((self._nq, self.n), np.float32)
        check(C.lib().spmv_solver_result_batch(self._h, out.ctypes.data), "spmv_solver_result_batch")
        return out

    def result(self):
        a = np.zeros(max(self.n, 1), np.float32)
        b = np.zeros(max(self.n, 1), np.float32)
        check(C.lib().spmv_solver_result(self._h, a.ctypes.data, b.ctypes.data), "spmv_solver_result")
        if self.algo == "hits":
            return a[: self.n], b[: self.n]
        return a[: self.n]

    def stats(self) -> dict:
        s = C.PlanStats()
        check(C.lib().spmv_solver_plan_stats(self._h, ctypes.byref(s)), "spmv_solver_plan_stats")
        return _stats_dict(s)

    def set_stop(self, tol: float = 1e-6, max_iter: int = 1000, fixed_iters: int = 0):
        """Change the stopping rule for the next runs (spmv_solver_set_stop); the plan stays."""
        check(C.lib().spmv_solver_set_stop(self._h, float(tol), int(max_iter), int(fixed_iters)),
              "spmv_solver_set_stop")

    @property
    def launches_per_iter(self) -> int:
        return int(C.lib().spmv_solver_launches_per_iter(self._h))

    def close(self):
        if getattr(self, "_h", None):
            C.lib().spmv_solver_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def pagerank(n, row_ptr, col, device=0, **kw):
    s = Solver("pagerank", n, row_ptr, col, device=device, iter_kw=kw.pop("iter_kw", None), **kw)
    info = s.run()
    return s.result(), info


def hits(n, row_ptr, col, device=0, **kw):
    s = Solver("hits", n, row_ptr, col, device=device, iter_kw=kw.pop("iter_kw", None), **kw)
    info = s.run()
    a, h = s.result()
    return a, h, info


def rwr(n, row_ptr, col, query, device=0, **kw):
    s = Solver("rwr", n, row_ptr, col, device=device, iter_kw=kw.pop("iter_kw", None), **kw)
    info = s.run(query)
    return s.result(), info


def bitonic_partition(row_len, P: int) -> np.ndarray:
    rl = _np(row_len, np.int64)
    owner = np.zeros(max(len(rl), 1), np.int32)
    check(C.lib().bitonic_partition(len(rl), _ptr(rl), int(P), owner.ctypes.data), "bitonic_partition")
    return owner[: len(rl)]


def partition_plan(row_len, P: int):
    """(owner, local_index, slot_rows) of the row-partitioned path (spmv_partition_plan)."""
    rl = _np(row_len, np.int64)
    owner = np.zeros(max(len(rl), 1), np.int32)
    lidx = np.zeros(max(len(rl), 1), np.int64)
    S = ctypes.c_int64(0)
    check(C.lib().spmv_partition_plan(len(rl), _ptr(rl), int(P), owner.ctypes.data, lidx.ctypes.data,
                                      ctypes.byref(S)), "spmv_partition_plan")
    return owner[: len(rl)], lidx[: len(rl)], int(S.value)


def needed_lists(row_ptr, col, owner, P: int, rank: int):
    """(send, recv): per peer q, the ascending vertex ids `rank` sends to / receives from q in the
    needed-columns exchange of the iteration matrix (row_ptr, col) under `owner` (spmv_needed_lists)."""
    rp = _np(row_ptr, np.int64)
    cl = _np(col, np.int32)
    ow = _np(owner, np.int32)
    n = len(rp) - 1
    sc = np.zeros(P, np.int64)
    rc = np.zeros(P, np.int64)
    check(C.lib().spmv_needed_lists(n, _ptr(rp), _ptr(cl), _ptr(ow), int(P), int(rank), sc.ctypes.data,
                                    rc.ctypes.data, None, None), "spmv_needed_lists")
    si = np.zeros(max(int(sc.sum()), 1), np.int32)
    ri = np.zeros(max(int(rc.sum()), 1), np.int32)
    check(C.lib().spmv_needed_lists(n, _ptr(rp), _ptr(cl), _ptr(ow), int(P), int(rank), sc.ctypes.data,
                                    rc.ctypes.data, si.ctypes.data, ri.ctypes.data), "spmv_needed_lists")
    so = np.concatenate([[0], np.cumsum(sc)])
    ro = np.concatenate([[0], np.cumsum(rc)])
    return ([si[so[q]:so[q + 1]] for q in range(P)], [ri[ro[q]:ro[q + 1]] for q in range(P)])


class Comm:
    """NCCL communicator for the row-partitioned path (Sec. 3.2).  The 128-byte unique id is
    created on rank 0 and broadcast by the caller (e.g. over a torch process group)."""

    @staticmethod
    def unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        check(C.lib().spmv_comm_unique_id(buf), "spmv_comm_unique_id")
        return buf.raw

    @classmethod
    def from_torch(cls, device: int, group=None):
        """Bootstrap over an initialised torch.distributed process group: rank 0 draws the NCCL
        unique id, every rank receives it by broadcast."""
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        obj = [cls.unique_id() if (rank == 0 and world > 1) else b"\0" * 128]
        if world > 1:
            dist.broadcast_object_list(obj, src=0, group=group)
        return cls(rank, world, obj[0], device)

    def __init__(self, rank: int, world: int, uid: bytes, device: int, _handle=None):
        if _handle is not None:
            self._h = _handle
        else:
            buf = ctypes.create_string_buffer(bytes(uid), 128)
            h = ctypes.c_void_p()
            check(C.lib().spmv_comm_create(rank, world, buf, device, ctypes.byref(h)), "spmv_comm_create")
            self._h = h
        self.rank, self.world = rank, world

    @classmethod
    def loopback(cls, world: int, device: int = 0):
        """Test transport: `world` logical ranks on one device (spmv_comm_create_loopback); drive
        each returned communicator from its own thread."""
        arr = (ctypes.c_void_p * world)()
        check(C.lib().spmv_comm_create_loopback(world, device, arr), "spmv_comm_create_loopback")
        return [cls(r, world, b"", device, _handle=ctypes.c_void_p(arr[r])) for r in range(world)]

    @classmethod
    def slices(cls, world: int, device: int = 0):
        """`world` row slices of one solver on one device sharing one exchange buffer
        (spmv_comm_create_slices); drive each returned communicator from its own thread."""
        arr = (ctypes.c_void_p * world)()
        check(C.lib().spmv_comm_create_slices(world, device, arr), "spmv_comm_create_slices")
        return [cls(r, world, b"", device, _handle=ctypes.c_void_p(arr[r])) for r in range(world)]

    def close(self):
        if getattr(self, "_h", None):
            C.lib().spmv_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
