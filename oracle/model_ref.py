"""model_ref -- TEST INFRASTRUCTURE ONLY.  Literal transcription of the paper's auto-tuner and
performance model (Sec. 3.3, Appendix E), for exact comparison with the product's C++.

  pm_paper      Alg. 3 PM(T, WL) / Eq. 1-5
  partition     Alg. 2 Partition(T)
  tile_count    Alg. 1 (tile loop, lines 4-8)
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


def pm_packed(hist, WL, perf, max_act_warp, align=8, split=True, ell_h=32, orient=0):
    """B200 reading of Alg. 3: the same wave model (Eq. 1-5) charged over
    the workloads the format actually builds (the packing of Solution 3 / format_ref with row
    splitting, R21, and clipping, R13), each looked up at its padded shape.
    hist: [(row length, count)] with lengths descending.  perf(kind, w, h) -> slots/s.
    Returns seconds."""
    rows = []
    for length, count in hist:
        rows += [length] * count
    waves = []                                   # per wave: [sum perf, sum size, count]
    def add(kind, w, h, size):
        if not waves or waves[-1][2] == max_act_warp:
            waves.append([0.0, 0.0, 0])
        wv = waves[-1]
        wv[0] += perf(kind, max(w, 1), h)
        wv[1] += size
        wv[2] += 1
    i = 0
    while i < len(rows):
        w = rows[i]
        hq = max(1, WL // max(w, 1))
        if split and w > WL:
            c = 0
            while c * WL < w:
                wp = _rup(min(WL, w - c * WL), align)
                add("rm", wp, 1, wp)
                c += 1
            i += 1
        elif ((w > 0) if orient == 1 else (False if orient == 2 else w >= hq)):
            h = min(hq, len(rows) - i)
            wp = _rup(w, align)
            add("rm", wp, h, h * wp)
            i += h
        else:
            take = min(_rup(hq, ell_h), len(rows) - i)
            hs = _rup(take, ell_h)
            add("cm", w, hs, hs * w)
            i += take
    return sum(S / (P / c) for P, S, c in waves)
