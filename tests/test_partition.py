"""Row-partitioned (multi-GPU) host logic on CPU: the library's bitonic partition equals the
oracle's snake order (reading R25), the slot layout is consistent, and a world-2
gloo run of the exchange protocol (each rank computes its own rows, one allgather of the slots)
reproduces the single-process product."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import graphgen
import oracle
from oracle import partition_ref


@pytest.mark.parametrize("P", [1, 2, 3, 5, 8])
def test_bitonic_matches_oracle(P):
    from paper_1103_2405_b200 import bitonic_partition, partition_plan
    rng = np.random.default_rng(P)
    lens = rng.zipf(1.8, 2001).astype(np.int64)
    own = bitonic_partition(lens, P)
    assert own.tolist() == partition_ref.bitonic_partition(lens.tolist(), P)
    owner, lidx, S = partition_plan(lens, P)
    assert np.array_equal(owner, own)
    counts = np.bincount(owner, minlength=P)
    assert counts.max() - counts.min() <= 1 and S == counts.max()
    for r in range(P):                       # local index = rank of the row among its owner's rows
        rows = np.nonzero(owner == r)[0]
        assert np.array_equal(lidx[rows], np.arange(len(rows)))


def test_partition_errors():
    from paper_1103_2405_b200 import SpmvError, bitonic_partition
    with pytest.raises(SpmvError, match="ERANGE"):
        bitonic_partition([1, 2], 3)
    with pytest.raises(SpmvError, match="EINVAL"):
        bitonic_partition([1, 2], 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, result_dir):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1103_2405_b200 import partition_plan
    G = graphgen.make_graph("t_small")
    rp, col = graphgen.keys_to_csr(G.keys, G.n, transpose=True)      # PageRank matrix A^T
    rl = np.diff(rp)
    owner, lidx, S = partition_plan(rl, world)
    x = graphgen.uniform_f32(G.n, seed=3)
    # this rank's rows, computed locally (the oracle stands in for the local SpMV)
    mine = np.nonzero(owner == rank)[0]
    sub_rp = np.concatenate([[0], np.cumsum(rl[mine])]).astype(np.int64)
    sub_col = np.concatenate([col[rp[r]:rp[r + 1]] for r in mine]) if len(mine) else np.zeros(0, np.int32)
    y_loc, _ = oracle.spmv(sub_rp, sub_col, None, x)
    slot = np.zeros(S, np.float64)
    slot[lidx[mine]] = y_loc
    gathered = [torch.zeros(S, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(gathered, torch.from_numpy(slot))
    G_all = torch.cat(gathered).numpy()
    y = G_all[owner.astype(np.int64) * S + lidx]                     # gpos = owner * S + local
    np.save(os.path.join(result_dir, f"y{rank}.npy"), y)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_exchange_protocol(world, tmp_path):
    port = _free_port()
    mp.spawn(_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    G = graphgen.make_graph("t_small")
    rp, col = graphgen.keys_to_csr(G.keys, G.n, transpose=True)
    ref, _ = oracle.spmv(rp, col, None, graphgen.uniform_f32(G.n, seed=3))
    for r in range(world):
        y = np.load(tmp_path / f"y{r}.npy")
        assert np.array_equal(y, ref)          # every rank holds the identical full vector


def _worker_pagerank(rank, world, port, result_dir, iters):
    """The row-partitioned PageRank protocol of csrc/dist.cu in fp64: bitonic ownership; on each
    rank the rows whose column is non-empty (out-degree > 0) first, so the exchanged slot carries
    only those z values plus two fp64 partials (sum |dp|, dangling mass) summed in rank order."""
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1103_2405_b200 import partition_plan
    G = graphgen.make_graph("t_small")
    n, c = G.n, 0.85
    outdeg = np.diff(G.row_ptr)
    rp, col = graphgen.keys_to_csr(G.keys, n, transpose=True)       # M = A^T
    owner, _, _ = partition_plan(np.diff(rp), world)
    col_ne = outdeg > 0
    lrow = np.zeros(n, np.int64)
    cnt_ne = np.zeros(world, np.int64)
    for r in range(world):
        own = np.nonzero(owner == r)[0]
        ne, em = own[col_ne[own]], own[~col_ne[own]]
        lrow[ne] = np.arange(len(ne))
        lrow[em] = len(ne) + np.arange(len(em))
        cnt_ne[r] = len(ne)
    S = int(cnt_ne.max())
    slot = S + 2
    mine = np.nonzero(owner == rank)[0]
    mine = mine[np.argsort(lrow[mine])]
    sub_rp = np.concatenate([[0], np.cumsum(np.diff(rp)[mine])]).astype(np.int64)
    sub_col = np.concatenate([col[rp[r]:rp[r + 1]] for r in mine]) if len(mine) else np.zeros(0, np.int32)
    inv = np.where(outdeg[mine] > 0, 1.0 / np.maximum(outdeg[mine], 1), 0.0)
    gpos = np.where(col_ne, owner.astype(np.int64) * slot + lrow, -1)
    p = np.full(len(mine), 1.0 / n)

    def exchange(p, partials):
        buf = np.zeros(slot)
        k = int(cnt_ne[rank])
        buf[:k] = (p * inv)[:k]
        assert not (p * inv)[k:].any()                 # empty columns carry nothing
        buf[S:] = partials
        parts = [torch.zeros(slot, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(buf))
        Gb = torch.cat(parts).numpy()
        z = np.where(gpos >= 0, Gb[np.maximum(gpos, 0)], 0.0)
        tot = sum(Gb[r * slot + S: r * slot + S + 2] for r in range(world))   # rank order
        return z, tot

    dm0 = float(p[outdeg[mine] == 0].sum())
    z, tot = exchange(p, [0.0, dm0])
    D = tot[1]
    rows_of = np.repeat(np.arange(len(mine)), np.diff(sub_rp))
    for _ in range(iters):
        y = np.bincount(rows_of, weights=z[sub_col], minlength=len(mine))     # fp64 local SpMV
        pn = c * (y + D / n) + (1 - c) / n
        part = [float(np.abs(pn - p).sum()), float(pn[outdeg[mine] == 0].sum())]
        p = pn
        z, tot = exchange(p, part)
        D = tot[1]
    # result gather (full slots)
    full = np.zeros(n)
    parts = [None] * world
    dist.all_gather_object(parts, (mine.tolist(), p.tolist()))
    for rows, vals in parts:
        full[rows] = vals
    np.save(os.path.join(result_dir, f"p{rank}.npy"), full)
    dist.destroy_process_group()


def test_gloo_pagerank_skip_empty_columns(tmp_path):
    world, iters = 2, 12
    port = _free_port()
    mp.spawn(_worker_pagerank, args=(world, port, str(tmp_path), iters), nprocs=world, join=True)
    G = graphgen.make_graph("t_small")
    ref, _ = oracle.pagerank(G.n, G.row_ptr, G.col, fixed_iters=iters)
    for r in range(world):
        p = np.load(tmp_path / f"p{r}.npy")
        assert np.abs(p - ref).sum() < 1e-12


# ---------------------------------------------------------------- needed-columns exchange (f3)

@pytest.mark.parametrize("P", [1, 2, 3, 5])
def test_needed_lists_brute_force(P):
    """spmv_needed_lists against a set computation: rank r sends to q exactly the vertices r owns
    that q's rows read, ascending; what r sends to q is what q expects from r."""
    from paper_1103_2405_b200 import needed_lists, partition_plan
    rp, col, _ = graphgen.random_csr(600, 600, 5000, seed=P, kind="powerlaw", valued=False)
    owner, _, _ = partition_plan(np.diff(rp), P)
    rows = np.repeat(np.arange(600), np.diff(rp))
    lists = [needed_lists(rp, col, owner, P, r) for r in range(P)]
    for r in range(P):
        send, recv = lists[r]
        for q in range(P):
            if q == r:
                assert len(send[q]) == 0 and len(recv[q]) == 0
                continue
            want_send = np.unique(col[(owner[rows] == q) & (owner[col] == r)])
            want_recv = np.unique(col[(owner[rows] == r) & (owner[col] == q)])
            assert np.array_equal(send[q], want_send) and np.array_equal(recv[q], want_recv)
            assert np.array_equal(send[q], lists[q][1][r])      # sender and receiver agree


def test_needed_lists_errors():
    from paper_1103_2405_b200 import SpmvError, needed_lists
    rp = np.array([0, 1, 2], np.int64)
    col = np.array([1, 0], np.int32)
    with pytest.raises(SpmvError):
        needed_lists(rp, col, np.array([0, 2], np.int32), 2, 0)     # owner out of range
    with pytest.raises(SpmvError):
        needed_lists(rp, col, np.array([0, 1], np.int32), 2, 2)     # rank out of range
    with pytest.raises(SpmvError):
        needed_lists(rp, np.array([1, 5], np.int32), np.array([0, 1], np.int32), 2, 0)


def _worker_pagerank_needed(rank, world, port, result_dir, iters):
    """The needed-columns protocol of csrc/dist.cu (exchange = 1) in fp64 over gloo point-to-point:
    each rank sends each peer the z values of the vertices on spmv_needed_lists' send list plus
    its two fp64 partials, and builds its x from its own z and the received segments."""
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1103_2405_b200 import needed_lists, partition_plan
    G = graphgen.make_graph("t_small")
    n, c = G.n, 0.85
    outdeg = np.diff(G.row_ptr)
    rp, col = graphgen.keys_to_csr(G.keys, n, transpose=True)       # M = A^T
    owner, _, _ = partition_plan(np.diff(rp), world)
    send, recv = needed_lists(rp, col, owner, world, rank)
    mine = np.nonzero(owner == rank)[0]
    rows = np.repeat(np.arange(n), np.diff(rp))
    sel = owner[rows] == rank
    inv_all = np.where(outdeg > 0, 1.0 / np.maximum(outdeg, 1), 0.0)
    p = np.zeros(n)
    p[mine] = 1.0 / n

    def exchange(p, partials):
        z = np.zeros(n)
        z[mine] = p[mine] * inv_all[mine]
        reqs, bufs = [], {}
        for q in range(world):
            if q == rank:
                continue
            out = torch.from_numpy(np.concatenate([z[send[q]], partials]))
            bufs[q] = torch.zeros(len(recv[q]) + 2, dtype=torch.float64)
            reqs.append(dist.isend(out, q))
            reqs.append(dist.irecv(bufs[q], q))
        for rq in reqs:
            rq.wait()
        tot = np.zeros(2)
        for q in range(world):                                       # rank order
            if q == rank:
                tot += partials
            else:
                b = bufs[q].numpy()
                z[recv[q]] = b[:len(recv[q])]
                tot += b[len(recv[q]):]
        return z, tot

    z, tot = exchange(p, np.array([0.0, float(p[mine][outdeg[mine] == 0].sum())]))
    D = tot[1]
    for _ in range(iters):
        y = np.bincount(rows[sel], weights=z[col[sel]], minlength=n)[mine]
        pn = c * (y + D / n) + (1 - c) / n
        part = np.array([float(np.abs(pn - p[mine]).sum()), float(pn[outdeg[mine] == 0].sum())])
        p[mine] = pn
        z, tot = exchange(p, part)
        D = tot[1]
    parts = [None] * world
    dist.all_gather_object(parts, (mine.tolist(), p[mine].tolist()))
    full = np.zeros(n)
    for rws, vals in parts:
        full[rws] = vals
    np.save(os.path.join(result_dir, f"p{rank}.npy"), full)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_pagerank_needed_exchange(world, tmp_path):
    iters = 12
    port = _free_port()
    mp.spawn(_worker_pagerank_needed, args=(world, port, str(tmp_path), iters), nprocs=world, join=True)
    G = graphgen.make_graph("t_small")
    ref, _ = oracle.pagerank(G.n, G.row_ptr, G.col, fixed_iters=iters)
    for r in range(world):
        p = np.load(tmp_path / f"p{r}.npy")
        assert np.abs(p - ref).sum() < 1e-12


def _worker_hits(rank, world, port, result_dir, iters, norm):
    """The row-partitioned HITS protocol of csrc/dist.cu in fp64: rows of the block matrix
    [[0, A^T], [A, 0]] dealt by the bitonic partition; every exchange carries the raw product y of
    a rank's rows plus its half sums and the L1 change of its previous normalisation; every rank
    sums the partials in rank order, normalises its own rows and the gathered x itself, and the
    stop decision lags one SpMV (reading R14: compared at the oracle's iteration count)."""
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1103_2405_b200 import partition_plan
    G = graphgen.make_graph("t_small")
    n = G.n
    src = np.repeat(np.arange(n), np.diff(G.row_ptr))
    dst = G.col.astype(np.int64)
    N = 2 * n
    # block rows: v < n (authority) reads h_u = x[n + u] for u -> v; n + u (hub) reads a_v = x[v]
    rows = np.concatenate([dst, n + src])
    cols = np.concatenate([n + src, dst])
    rl = np.bincount(rows, minlength=N)
    owner, _, _ = partition_plan(rl, world)
    mine = np.nonzero(owner == rank)[0]
    sel = owner[rows] == rank
    half = (np.arange(N) >= n).astype(np.int64)
    x = np.full(N, 1.0 / n)                      # a(0) = h(0) = 1/|V| (L440)
    v_old = np.full(N, 1.0 / n)
    res_own, it = 0.0, 0
    while True:
        y = np.bincount(rows[sel], weights=x[cols[sel]], minlength=N)[mine]      # own rows, raw
        d = np.abs(y) if norm == 1 else y * y
        part = np.array([d[half[mine] == 0].sum(), d[half[mine] == 1].sum(), res_own])
        slot = np.zeros(N)
        slot[mine] = y
        ys = [torch.zeros(N, dtype=torch.float64) for _ in range(world)]
        ps = [torch.zeros(3, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(ys, torch.from_numpy(slot))
        dist.all_gather(ps, torch.from_numpy(part))
        tot = np.zeros(3)
        for q in range(world):                                                   # rank order
            tot += ps[q].numpy()
        if it >= 1 and it >= iters:                                              # lagged stop
            break
        nrm = tot[:2] if norm == 1 else np.sqrt(tot[:2])
        yall = sum(t.numpy() for t in ys)
        scale = np.where(nrm[half] > 0, 1.0 / np.where(nrm[half] > 0, nrm[half], 1.0), 0.0)
        uni = 1.0 / n if norm == 1 else 1.0 / np.sqrt(n)
        x = np.where(nrm[half] > 0, yall * scale, uni)                          # gathered x, normalised
        v_new = x[mine]
        res_own = float(np.abs(v_new - v_old[mine]).sum())
        v_old[mine] = v_new
        it += 1
    parts = [None] * world
    dist.all_gather_object(parts, (mine.tolist(), v_old[mine].tolist()))
    full = np.zeros(N)
    for rws, vals in parts:
        full[rws] = vals
    np.save(os.path.join(result_dir, f"h{rank}.npy"), full)
    dist.destroy_process_group()


@pytest.mark.parametrize("world,norm", [(2, 1), (3, 2)])
def test_gloo_hits_protocol(world, norm, tmp_path):
    iters = 10
    port = _free_port()
    mp.spawn(_worker_hits, args=(world, port, str(tmp_path), iters, norm), nprocs=world, join=True)
    G = graphgen.make_graph("t_small")
    ra, rh, _ = oracle.hits(G.n, G.row_ptr, G.col, norm=norm, fixed_iters=iters)
    for r in range(world):
        v = np.load(tmp_path / f"h{r}.npy")
        assert np.abs(v[:G.n] - ra).sum() < 1e-12 and np.abs(v[G.n:] - rh).sum() < 1e-12


def _worker_rwr(rank, world, port, result_dir, iters, q):
    """The row-partitioned RWR protocol (Eq. 9, readings R6-R8) in fp64: rows of W = A_sym D^-1
    by the bitonic partition of A_sym's rows; each rank exchanges z = r / deg of its own vertices
    (allgather of slots) plus its L1 change; r' = c (A_sym z) + (1 - c) e_q on its own rows."""
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1103_2405_b200 import partition_plan
    G = graphgen.make_graph("t_small")
    n, c = G.n, 0.9
    u = np.repeat(np.arange(n), np.diff(G.row_ptr))
    v = G.col.astype(np.int64)
    key = np.unique(np.concatenate([u * n + v, v * n + u]))                   # A u A^T, merged
    rows, cols = key // n, key % n
    deg = np.bincount(rows, minlength=n).astype(np.float64)
    owner, _, _ = partition_plan(deg.astype(np.int64), world)
    mine = np.nonzero(owner == rank)[0]
    sel = owner[rows] == rank
    inv = np.where(deg > 0, 1.0 / np.maximum(deg, 1), 0.0)
    r = np.zeros(n)
    r[q] = 1.0                                                                # r(0) = e_q (R7)
    for _ in range(iters):
        slot = np.zeros(n)
        slot[mine] = r[mine] * inv[mine]
        zs = [torch.zeros(n, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(zs, torch.from_numpy(slot))
        z = sum(t.numpy() for t in zs)
        y = np.bincount(rows[sel], weights=z[cols[sel]], minlength=n)[mine]
        rn = c * y + (1 - c) * (mine == q)
        r[mine] = rn
    parts = [None] * world
    dist.all_gather_object(parts, (mine.tolist(), r[mine].tolist()))
    full = np.zeros(n)
    for rws, vals in parts:
        full[rws] = vals
    np.save(os.path.join(result_dir, f"r{rank}.npy"), full)
    dist.destroy_process_group()


def test_gloo_rwr_protocol(tmp_path):
    world, iters = 2, 15
    G = graphgen.make_graph("t_small")
    q = int(np.nonzero(np.diff(G.row_ptr) > 0)[0][3])
    port = _free_port()
    mp.spawn(_worker_rwr, args=(world, port, str(tmp_path), iters, q), nprocs=world, join=True)
    ref, _ = oracle.rwr(G.n, G.row_ptr, G.col, q, fixed_iters=iters)
    for rk in range(world):
        assert np.abs(np.load(tmp_path / f"r{rk}.npy") - ref).sum() < 1e-12


def test_grid_volume_brute_force():
    """bench/exchange_volume.grid_volume (the 2-D partition of P:L106-L108) against a set
    computation on a small graph: x values each rank's columns need from other owners plus the
    partial-y rows it sends to other owners."""
    import importlib.util
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("ev", os.path.join(root, "bench", "exchange_volume.py"))
    ev = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(ev)
    rp, col, _ = graphgen.random_csr(300, 300, 3000, seed=4, kind="powerlaw", valued=False)
    for P in (2, 4, 6, 8):
        owner = np.random.default_rng(P).integers(0, P, 300).astype(np.int32)
        got, shape = ev.grid_volume(rp, col, owner, P)
        pr, pc = map(int, shape.split("x"))
        xs, ys = set(), set()
        for v in range(300):
            for u in col[rp[v]:rp[v + 1]]:
                h = (owner[v] // pc) * pc + owner[u] % pc
                if owner[u] != h:
                    xs.add((h, int(u)))
                if owner[v] != h:
                    ys.add((h, v))
        assert got == len(xs) + len(ys) and pr * pc == P
