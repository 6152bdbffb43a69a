"""The device generator (graphgen/graphgen_gpu.cu) against the host generator (graphgen.c).

Input infrastructure, not the method: the keys must be bit-identical to the host's (same
counter-based draws, rounds, thinning and relabel), and a rank's rows of each iteration matrix must
equal the rows numpy builds from the host keys."""
import numpy as np
import pytest

import graphgen

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("config", ["t_small", "c1", "t_mid", "c2"])
def test_device_keys_equal_host(gpu, config):
    host = graphgen.make_graph(config)
    dg = graphgen.DeviceGraph(config, device=gpu)
    try:
        assert dg.m == host.m
        assert np.array_equal(dg.keys(), host.keys)
        od, idg = dg.degrees()
        u = (host.keys >> np.uint64(32)).astype(np.int64)
        v = (host.keys & np.uint64(0xFFFFFFFF)).astype(np.int64)
        assert np.array_equal(od, np.bincount(u, minlength=host.n))
        assert np.array_equal(idg, np.bincount(v, minlength=host.n))
    finally:
        dg.close()


def _rows_ref(keys, n, kind, ids):
    u = (keys >> np.uint64(32)).astype(np.int64)
    v = (keys & np.uint64(0xFFFFFFFF)).astype(np.int64)
    if kind == graphgen.KIND_A:
        r, c = u, v
    elif kind == graphgen.KIND_AT:
        r, c = v, u
    else:
        r = np.concatenate([v, n + u])
        c = np.concatenate([n + u, v])
    o = np.lexsort((c, r))
    r, c = r[o], c[o]
    sel = np.isin(r, ids)
    r, c = r[sel], c[sel]
    rp = np.zeros(len(ids) + 1, dtype=np.int64)
    pos = np.searchsorted(ids, r)
    np.add.at(rp, pos + 1, 1)
    return np.cumsum(rp), c.astype(np.int32)


@pytest.mark.parametrize("kind", [graphgen.KIND_A, graphgen.KIND_AT, graphgen.KIND_HITS])
@pytest.mark.parametrize("P", [1, 3])
def test_owned_rows(gpu, kind, P):
    host = graphgen.make_graph("t_mid")
    dg = graphgen.DeviceGraph("t_mid", device=gpu)
    try:
        N = 2 * host.n if kind == graphgen.KIND_HITS else host.n
        owner = (np.arange(N) * 7919 % P).astype(np.int32)     # scattered ownership
        seen = 0
        for q in range(P):
            ids, rp, col = dg.owned_rows(kind, owner, q)
            assert np.array_equal(ids, np.nonzero(owner == q)[0])
            rp_ref, col_ref = _rows_ref(host.keys, host.n, kind, ids)
            assert np.array_equal(rp, rp_ref)
            assert np.array_equal(col, col_ref)
            seen += len(col)
        assert seen == (2 * host.m if kind == graphgen.KIND_HITS else host.m)
    finally:
        dg.close()
