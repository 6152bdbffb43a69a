"""The product's performance model / auto-tuner against the oracle's transcription
(oracle/model_ref.py) under a fixed offline table: per-tile predicted time equal to the
transcription, and the auto-tuned WL the argmin of an independent re-enumeration (Alg. 2)."""
import json
import math

import numpy as np
import pytest

import graphgen
from oracle import format_ref, model_ref

PERF = {"rm": 1.0e9, "cm": 2.5e9}          # constant per kind: lookup is exact, waves matter
TABLE = dict(version=1, max_act_warp=96, launch_us=3.0, stage_GBps=5000.0, rmw_GBps=2500.0)


def write_table(tmp_path, **extra):
    ent = []
    for cached in (0, 1):
        for valued in (0, 1):
            for w in (1, 8, 64, 4096):
                for h in (1, 32, 1024):
                    ent.append([cached, valued, 0, w, h, PERF["rm"]])
                    ent.append([cached, valued, 1, w, h, PERF["cm"]])
    path = tmp_path / "table.json"
    path.write_text(json.dumps(dict(TABLE, entries=ent, **extra)))
    return str(path)


def tile_hists(n_rows, n_cols, rp, col, tw, T):
    collen, perm, inv = format_ref.column_order(n_cols, col)
    hists = [dict() for _ in range(T + 1)]
    total = np.diff(rp)
    for i in range(n_rows):
        seg = np.zeros(T + 1, np.int64)
        for k in inv[col[rp[i]:rp[i + 1]]]:
            t = k // tw
            seg[min(t, T)] += 1
        for t in range(T + 1):
            if seg[t] or (t == T and total[i] == 0):
                hists[t][seg[t]] = hists[t].get(seg[t], 0) + 1
    return [sorted(h.items(), key=lambda kv: -kv[0]) for h in hists]


def expected_us(h, WL, t, T, tw, cached, split=True, tail_frac=0.0, orient=0):
    # the oracle's per-tile prediction (pinned by hand in tests/test_oracle_pins.py)
    return model_ref.tile_time_us(h, WL, lambda k, w, hh: PERF[k], TABLE["max_act_warp"], tile_index=t,
                                  tile_width=tw, cached=cached, launch_us=TABLE["launch_us"],
                                  stage_GBps=TABLE["stage_GBps"], rmw_GBps=TABLE["rmw_GBps"],
                                  tail_frac=tail_frac, split=split, orient=orient)


@pytest.mark.parametrize("seed,tail,orient", [(0, 0.0, 0), (1, 0.0, 0), (2, 0.0, 0), (3, 0.0, 0), (4, 0.5, 0),
                                              (5, 0.5, 0), (6, 0.0, 1), (7, 0.5, 2), (8, 0.0, 3), (9, 0.5, 3)])
def test_predicted_time_equals_transcription(seed, tail, orient, tmp_path):
    from paper_1103_2405_b200 import Plan
    table = write_table(tmp_path, tail_frac=tail)
    rng = np.random.default_rng(seed)
    nr, nc = int(rng.integers(200, 800)), int(rng.integers(200, 800))
    rp, col, _ = graphgen.random_csr(nr, nc, int(rng.integers(2000, 20000)), seed=seed, kind="powerlaw", valued=False)
    tw, T = 64, 3
    wls = [int(x) for x in rng.choice([32, 64, 128, 256], size=T + 1)]
    p = Plan(nr, nc, rp, col, None, device=-1, tile_width=tw, num_tiles=T, workload_sizes=wls,
             perf_table_path=table, orient=orient)
    st = p.stats()
    assert st["perf_table_loaded"]
    hists = tile_hists(nr, nc, rp, col, tw, T)
    for t in range(T + 1):
        o_t = 0 if (orient == 3 and t == T) else orient      # TILE-COO: composite remainder
        exp = expected_us(hists[t], wls[t], t, T, tw, cached=t < T, tail_frac=tail, orient=o_t)
        assert math.isclose(st["tile_predicted_us"][t], exp, rel_tol=1e-9), (t, st["tile_predicted_us"][t], exp)


def test_autotuned_wl_is_argmin(tmp_path):
    """Alg. 2 (B200 candidates, reading R21): the chosen WL minimises the model over the powers of
    two and the multiples of the longest row up to max(longest, 32768) (strict <, R22)."""
    from paper_1103_2405_b200 import Plan
    table = write_table(tmp_path)
    G = graphgen.make_graph("t_small")
    rp, col = graphgen.keys_to_csr(G.keys, G.n, transpose=True)
    tw, T = 256, 2
    p = Plan(G.n, G.n, rp, col, None, device=-1, tile_width=tw, num_tiles=T, perf_table_path=table)
    st = p.stats()
    hists = tile_hists(G.n, G.n, rp, col, tw, T)
    for t in range(T + 1):
        cands = model_ref.b200_candidates(hists[t][0][0] if hists[t] else 1)
        times = [model_ref.pm_packed(hists[t], c, lambda k, w, h: PERF[k], TABLE["max_act_warp"]) for c in cands]
        best = cands[int(np.argmin(times))]       # argmin keeps the first (smallest) on ties
        assert st["wl"][t] == best, (t, st["wl"][t], best, times)


def test_eq1_waves_in_product(tmp_path):
    """2000 one-slot workloads with MAX_ACT_WARP = 960 form ceil(2000/960) = 3 waves (Eq. 1,
    L124): with a uniform table the predicted time is the padded size, independent of waves."""
    from paper_1103_2405_b200 import Plan
    ent = [[c, v, k, w, h, 1e9] for c in (0, 1) for v in (0, 1) for k in (0, 1) for w in (1, 4096) for h in (1, 1024)]
    path = tmp_path / "u.json"
    path.write_text(json.dumps(dict(TABLE, max_act_warp=960, entries=ent)))
    n = 2000
    rp = np.arange(n + 1)
    col = np.arange(n, dtype=np.int32)
    p = Plan(n, n, rp, col, None, device=-1, tile_width=n, num_tiles=0, workload_sizes=[1],
             align_rm=8, perf_table_path=str(path))
    # WL=1, rows of length 1: w=1 >= hq=1 -> row major, padded to 8 slots; 2000 workloads
    us = p.stats()["tile_predicted_us"][0]
    assert math.isclose(us, 2000 * 8 / 1e9 * 1e6 + TABLE["launch_us"], rel_tol=1e-12)


# per x regime constants (mode: (rm, cm) slots/s): 0 uncached uniform, 1 staged, 2 hub tile, 3 beyond L2
PERF_MODE = {0: (1.0e9, 2.5e9), 1: (3.0e9, 4.0e9), 2: (1.5e9, 2.0e9), 3: (0.4e9, 0.7e9)}


@pytest.mark.parametrize("stage,budget", [(1, 200.0), (0, 200.0), (1, 1e9), (0, 1e9)])
def test_x_regime_per_tile(stage, budget, tmp_path):
    """Reading R32: tile t's table regime is 1 when staged; otherwise 3 when its x span (tw or
    the remainder's columns, 4 bytes each) exceeds the L2 budget, 2 for the first tile, else 0.
    Per-tile predicted time equals the transcription with that regime's table."""
    from paper_1103_2405_b200 import Plan
    ent = []
    for mode, (prm, pcm) in PERF_MODE.items():
        for valued in (0, 1):
            for w in (1, 8, 64, 4096):
                for h in (1, 32, 1024):
                    ent += [[mode, valued, 0, w, h, prm], [mode, valued, 1, w, h, pcm]]
    path = tmp_path / "modes.json"
    path.write_text(json.dumps(dict(TABLE, l2_budget_bytes=budget, entries=ent)))
    rp, col, _ = graphgen.random_csr(500, 700, 9000, seed=11, kind="powerlaw", valued=False)
    tw, T, wl = 64, 3, 128
    p = Plan(500, 700, rp, col, None, device=-1, tile_width=tw, num_tiles=T, workload_size=wl,
             perf_table_path=str(path), stage_x=stage)
    st = p.stats()
    hists = tile_hists(500, 700, rp, col, tw, T)
    for t in range(T + 1):
        span = tw if t < T else 700 - T * tw
        cached = bool(stage) and t < T
        mode = 1 if cached else (3 if span * 4.0 > budget else (2 if t == 0 else 0))
        prm, pcm = PERF_MODE[mode]
        us = model_ref.tile_time_us(hists[t], wl, lambda k, w, h: prm if k == "rm" else pcm,
                                    TABLE["max_act_warp"], tile_index=t, tile_width=tw, cached=cached,
                                    launch_us=TABLE["launch_us"], stage_GBps=TABLE["stage_GBps"],
                                    rmw_GBps=TABLE["rmw_GBps"])
        assert math.isclose(st["tile_predicted_us"][t], us, rel_tol=1e-9), (t, mode, st["tile_predicted_us"][t], us)


def test_model_chooses_orientation(tmp_path):
    """orient = -1: the plan takes the orientation (composite, CSR-vector, ELL, TILE-COO)
    with the smallest predicted time; its prediction equals that orientation's own plan's."""
    from paper_1103_2405_b200 import Plan
    table = write_table(tmp_path)
    rp, col, _ = graphgen.random_csr(3000, 3000, 60000, seed=7, kind="powerlaw", valued=False)
    pred = {}
    for o in (0, 1, 2, 3):
        st = Plan(3000, 3000, rp, col, None, device=-1, orient=o, perf_table_path=table, two_phase=0).stats()
        pred[o] = st["predicted_us"]
        assert st["orient"] == o
    st = Plan(3000, 3000, rp, col, None, device=-1, orient=-1, perf_table_path=table, two_phase=0).stats()
    best = min(pred, key=lambda o: (pred[o], o))
    assert st["orient"] == best and math.isclose(st["predicted_us"], pred[best], rel_tol=1e-12), (pred, st["orient"])
