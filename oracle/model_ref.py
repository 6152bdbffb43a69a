"""model_ref -- TEST INFRASTRUCTURE ONLY.  Literal transcription of the paper's auto-tuner and
performance model (Sec. 3.3, Appendix E), for exact comparison with the product's C++.

  pm_paper      Alg. 3 PM(T, WL) / Eq. 1-5
  partition     Alg. 2 Partition(T)
  tile_count    Alg. 1 (tile loop, lines 4-8)
  pm_packed     Alg. 3 / Eq. 1-5 over the B200 packing (packed_workloads, wave_time)
  tile_time_us  pm_packed + the B200 per-launch terms (launch, staging, y RMW, tail R31)
Pins (tests/test_oracle_pins.py): pm_paper by Eq. 1's anchor and a hand-traced total;
pm_packed equal to pm_paper in paper mode up to the clipped slots, and by two hand-traced B200
packings; tile_time_us by hand-computed terms.
Readings: R20 (table entry = whole-GPU slots/s at shape (w,h); Size counts padded slots;
P_i unweighted mean), R22 (strict <, smallest WL wins ties), R23 (sum over every realised wave),
R21 paper mode (empty candidate set -> WL_low).
"""
from __future__ import annotations

import math


def padding(w: int, h: int, warp: int = 32):
    """Alg. 3 line 10: pad w (row major, w >= h) or h (column major) to a warp multiple."""
    if w >= h:
        return ((w + warp - 1) // warp) * warp, h
    return w, ((h + warp - 1) // warp) * warp


def pm_paper(row_len, WL: int, perf, max_act_warp: int, warp: int = 32):
    """Alg. 3.  row_len: the tile's row lengths sorted high to low (non-empty rows).
    perf(w, h) -> throughput (padded slots per second, whole GPU).  Returns (total, detail)."""
    nnz = sum(row_len)
    n_warp = math.ceil(nnz / WL)                       # line 3
    I = math.ceil(n_warp / max_act_warp)               # line 5, Eq. 1
    P, Size, Cnt = {}, {}, {}
    i = j = 0                                          # line 6
    while i < len(row_len):                            # line 7
        w = row_len[i]                                 # line 9
        h = WL // w
        w, h = padding(w, h, warp)                     # line 10
        it = j // max_act_warp                         # line 11
        P[it] = P.get(it, 0.0) + perf(w, h)            # line 12
        Size[it] = Size.get(it, 0) + w * h             # line 13, Eq. 4
        Cnt[it] = Cnt.get(it, 0) + 1                   # line 14
        j += 1                                         # line 15
        i += h
    total = 0.0
    t = {}
    for it in sorted(P):                               # lines 17-20 (R23: every realised wave)
        Pm = P[it] / Cnt[it]                           # Eq. 5
        t[it] = Size[it] / Pm                          # Eq. 3
        total += t[it]                                 # Eq. 2
    return total, dict(n_warp=n_warp, I=I, waves=len(P), t=t, size=Size, cnt=Cnt)


def partition(row_len, perf, max_act_warp: int, warp: int = 32):
    """Alg. 2: WL from WL_low = RowLength[0] in steps of RowLength[0] while WL <= WL_up =
    floor(NNZ / MAX_ACT_WARP); argmin of PM with strict <.  Empty set -> WL_low (R21)."""
    L = row_len[0]
    wl_up = sum(row_len) // max_act_warp
    opt_wl, opt_time = 0, math.inf
    wl = L
    while wl <= wl_up:
        tm, _ = pm_paper(row_len, wl, perf, max_act_warp, warp)
        if tm < opt_time:
            opt_time, opt_wl = tm, wl
        wl += L
    if opt_wl == 0:
        opt_wl = L
        opt_time, _ = pm_paper(row_len, L, perf, max_act_warp, warp)
    return opt_wl, opt_time


def b200_candidates(longest: int, cap: int = 32768, limit: int = 96):
    """Reading R21 (B200 mode, rows longer than WL split): the candidate WLs of Alg. 2 are the
    powers of two from 32 up and the multiples of the longest row, both up to
    max(longest, cap) (cap: the table bound); at most `limit` multiples."""
    L = max(1, longest)
    up = max(L, cap)
    c = set()
    v = 32
    while v <= up:
        c.add(v)
        v *= 2
    k = L
    n = 0
    while k <= up and n < limit:
        c.add(k)
        k += L
        n += 1
    return sorted(c)


def tile_count(collen_sorted, n_cols: int, tile_width: int) -> int:
    """Alg. 1 lines 3-8 with reading R10 (continue while NTile*TW < n)."""
    nt = 0
    while nt * tile_width < n_cols:
        if collen_sorted[nt * tile_width] <= 1:
            break
        nt += 1
    return nt


def _rup(a, b):
    return (a + b - 1) // b * b


def packed_workloads(hist, WL, align=8, split=True, ell_h=32, orient=0):
    """The workloads the B200 packing walk forms over a tile (Solution 3 P:L88 with Alg. 3's
    partition lines 8-15, reading R12; row splitting R21; clipping of the last workload R13):
    a list of (kind, padded w, padded h, padded slots).  hist: [(row length, count)], lengths
    descending."""
    rows = []
    for length, count in hist:
        rows += [length] * count
    out = []
    i = 0
    while i < len(rows):
        w = rows[i]
        hq = max(1, WL // max(w, 1))
        if orient == 3 and not (split and w > WL):
            # TILE-COO (dense tiles): whole rows while at most WL entries (at least one),
            # padded to 32 slots; charged at the row-major table shape (slots, 1)
            h, tot = 0, 0
            while i + h < len(rows) and (h == 0 or tot + rows[i + h] <= WL):
                tot += rows[i + h]
                h += 1
            wp = _rup(tot, 32)
            out.append(("rm", wp, 1, wp))
            i += h
            continue
        if split and w > WL:
            c = 0
            while c * WL < w:
                wp = _rup(min(WL, w - c * WL), align)
                out.append(("rm", wp, 1, wp))
                c += 1
            i += 1
        elif ((w > 0) if orient == 1 else (False if orient == 2 else w >= hq)):   # orient 3: composite here
            h = min(hq, len(rows) - i)
            wp = _rup(w, align)
            out.append(("rm", wp, h, h * wp))
            i += h
        else:
            take = min(_rup(hq, ell_h), len(rows) - i)
            hs = _rup(take, ell_h)
            out.append(("cm", w, hs, hs * w))
            i += take
    return out


def wave_time(workloads, perf, max_act_warp):
    """Eq. 1-5 over a workload sequence: consecutive groups of MAX_ACT_WARP workloads form the
    waves (Alg. 3 line 11), t_i = Size_i / mean P_i (Eq. 3-5), summed over every realised wave
    (Eq. 2, R23).  perf(kind, w, h) -> slots/s."""
    total = 0.0
    for s in range(0, len(workloads), max_act_warp):
        wave = workloads[s:s + max_act_warp]
        P = sum(perf(k, max(w, 1), h) for k, w, h, _ in wave)
        S = sum(size for *_, size in wave)
        total += S / (P / len(wave))
    return total


def pm_packed(hist, WL, perf, max_act_warp, align=8, split=True, ell_h=32, orient=0):
    """B200 reading of Alg. 3: the same wave model (Eq. 1-5) charged over
    the workloads the format actually builds (packed_workloads), each looked up at its padded
    shape.  Returns seconds."""
    return wave_time(packed_workloads(hist, WL, align, split, ell_h, orient), perf, max_act_warp)


def tile_time_us(hist, WL, perf, max_act_warp, *, tile_index, tile_width, cached, launch_us,
                 stage_GBps, rmw_GBps, tail_frac=0.0, sm_count=148, align=8, split=True, ell_h=32,
                 orient=0):
    """Per-tile predicted time in microseconds: pm_packed plus the B200 terms the paper's model
    does not carry (P:L220 names them qualitatively; R31):
      launch      launch_us per non-empty tile ("restart a kernel for each tile");
      staging     cached tiles copy their x segment into every SM: tile_width * 4 B * sm_count
                  at stage_GBps;
      y RMW       tiles after the first read and write 8 B per touched row at rmw_GBps;
      tail (R31)  tail_frac of one workload's duration under load, WL / (mean P / MAX_ACT_WARP).
    An empty tile costs nothing."""
    wls = packed_workloads(hist, WL, align, split, ell_h, orient)
    rows = sum(c for _, c in hist)
    if not rows:
        return 0.0
    sec = wave_time(wls, perf, max_act_warp)
    if tail_frac and wls:
        mean_perf = sum(perf(k, max(w, 1), h) for k, w, h, _ in wls) / len(wls)
        sec += tail_frac * WL * max_act_warp / mean_perf
    us = sec * 1e6 + launch_us
    if cached:
        us += tile_width * 4.0 * sm_count / (stage_GBps * 1e3)
    if tile_index > 0:
        us += rows * 8.0 / (rmw_GBps * 1e3)
    return us
