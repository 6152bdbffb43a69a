"""format_ref -- TEST INFRASTRUCTURE ONLY.  Independent re-implementation of the tiled-composite
layout, written from the paper, for byte-for-byte comparison with the
product builder's exported arrays.  Shares no code with paper_1103_2405_b200/.

Follows, step by step:
  a1/a2  column lengths, reorder columns by decreasing length     Solution 2, PAPER.md L66, L68
  a3     fixed-width column tiles + one remainder tile            Solution 1, L56-L60; L90-L92
  a4     rows of each tile ranked by in-tile length, high to low  Solution 3, L86-L88
  a5     rows packed into ~WL workloads; w >= h -> row major,
         else column major; pads to warp multiples               Solution 3, L88, L94; Alg. 3
Readings: R9 entries kept as given; R12 Alg. 3's h = floor(WL/w); R13 padding and
clipping; R15 ties by ascending id; R16 sentinel column; R17 camping pad; R18 align_rm;
R19 composite remainder; R21 split of rows longer than WL.

This is plain Python over rows; use it at sizes up to ~1e6 entries.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

KIND_RM, KIND_CM, KIND_SPLIT, KIND_COO = 0, 1, 2, 3
COO_END = 1 << 31          # TILE-COO: flags the last entry of each row in its column word
FLAG_ACC = 1 << 29       # row already written by an earlier tile: add instead of store
FLAG_FINAL = 1 << 30     # no later tile touches this row: its value is final after this write
PAD_ROW = 0xFFFFFFFF     # padding row of a column-major slab (no write)


def _roundup(a: int, b: int) -> int:
    return ((a + b - 1) // b) * b


@dataclass
class Layout:
    n_rows: int
    n_cols: int
    pattern: bool
    perm: np.ndarray            # int32 [n_cols]: relabelled position k -> original column
    inv: np.ndarray             # int32 [n_cols]: original column j -> relabelled position
    tiles: np.ndarray           # int64 [T+1, 4]: col_lo, col_hi, wl_begin, wl_end
    desc: dict                  # per-workload arrays: off, row_base, w, h, kind, kvec, split_id, chunk
    row_id: np.ndarray          # uint32: row | FLAG_ACC | FLAG_FINAL, or PAD_ROW
    slot_col: np.ndarray        # int32: tile-relative column; sentinel = tile width
    slot_val: np.ndarray | None # float32 (None for pattern)
    split: np.ndarray           # int32 [n_split, 3]: row entry, n_chunks, partial_base
    meta: dict = field(default_factory=dict)


def column_order(n_cols: int, col: np.ndarray):
    """a1/a2: collen[j] = entries in column j; columns ordered by (length desc, id asc)."""
    collen = np.zeros(n_cols, dtype=np.int64)
    for j in col.tolist():
        collen[j] += 1
    order = sorted(range(n_cols), key=lambda j: (-int(collen[j]), j))
    perm = np.array(order, dtype=np.int32)
    inv = np.zeros(n_cols, dtype=np.int32)
    for k, j in enumerate(order):
        inv[j] = k
    return collen, perm, inv


def paper_tile_count(collen_sorted: np.ndarray, n_cols: int, tw: int) -> int:
    """Alg. 1: add tiles of TW columns while the tile's first column has
    >= 2 entries; loop while NTile*TW < n (reading R10: ceil)."""
    t = 0
    while t * tw < n_cols:
        if collen_sorted[t * tw] <= 1:
            break
        t += 1
    return t


def build(n_rows, n_cols, row_ptr, col, val, tile_width, num_tiles, workload_sizes,
          align_rm=8, split_long_rows=True, camping_pad=False, ell_h=32, orient=0) -> Layout:
    """Build the layout from explicit parameters (the autotuner is not involved here).
    workload_sizes: list of num_tiles + 1 ints (the last is the remainder tile's WL)."""
    row_ptr = np.asarray(row_ptr, dtype=np.int64)
    col = np.asarray(col, dtype=np.int32)
    pattern = val is None
    if not pattern:
        val = np.asarray(val, dtype=np.float32)
    T = int(num_tiles)
    assert len(workload_sizes) == T + 1
    collen, perm, inv = column_order(n_cols, col)

    # a3: tile column ranges; tile T is the remainder [min(T*TW, n), n)
    ranges = []
    for t in range(T):
        lo = t * tile_width
        ranges.append((lo, min(lo + tile_width, n_cols)))
    ranges.append((min(T * tile_width, n_cols), n_cols))

    def tile_of(k):  # relabelled column -> tile index
        for t, (lo, hi) in enumerate(ranges):
            if lo <= k < hi:
                return t
        raise AssertionError

    # a4: per (tile, row) the in-tile entries ordered by (relabelled column asc, position asc)
    per_tile = [dict() for _ in range(T + 1)]
    total_len = np.zeros(n_rows, dtype=np.int64)
    for i in range(n_rows):
        ents = []
        for p in range(int(row_ptr[i]), int(row_ptr[i + 1])):
            k = int(inv[col[p]])
            ents.append((k, p))
        ents.sort()
        total_len[i] = len(ents)
        for k, p in ents:
            t = tile_of(k)
            per_tile[t].setdefault(i, []).append((k - ranges[t][0], None if pattern else val[p]))
    touched = [set(per_tile[t].keys()) for t in range(T + 1)]
    zero_rows = [i for i in range(n_rows) if total_len[i] == 0]

    desc = {k: [] for k in ("off", "row_base", "w", "h", "kind", "kvec", "split_id", "chunk")}
    row_id, slot_col, slot_val, split = [], [], [], []
    tiles = np.zeros((T + 1, 4), dtype=np.int64)

    def flags_for(t, i):
        f = i
        if any(i in touched[s] for s in range(t)):
            f |= FLAG_ACC
        if not any(i in touched[s] for s in range(t + 1, T + 1)):
            f |= FLAG_FINAL
        return f

    def emit(off, rb, w, h, kind, kvec, sid, ch):
        for k_, v_ in zip(("off", "row_base", "w", "h", "kind", "kvec", "split_id", "chunk"),
                          (off, rb, w, h, kind, kvec, sid, ch)):
            desc[k_].append(v_)

    def camp():
        nonlocal slot_col, slot_val
        size = len(slot_col) - cur_off
        if camping_pad and size > 0 and size % 512 == 0:
            slot_col.extend([sentinel] * 64)
            if not pattern:
                slot_val.extend([np.float32(0)] * 64)

    for t in range(T + 1):
        lo, hi = ranges[t]
        sentinel = hi - lo
        WL = int(workload_sizes[t])
        assert WL >= 1
        rows = sorted(per_tile[t].keys(), key=lambda i: (-len(per_tile[t][i]), i))
        if t == T:
            rows = rows + zero_rows       # length-0 rows sort last, by id (R15)
        lens = [len(per_tile[t].get(i, [])) for i in rows]
        tiles[t, 0], tiles[t, 1] = lo, hi
        tiles[t, 2] = len(desc["off"])
        i = 0
        coo = orient == 3 and t < T               # TILE-COO: COO dense tiles
        orient_t = 0 if orient == 3 else orient   # ... and a composite remainder (R19)
        while i < len(rows):
            w = lens[i]
            hq = max(1, WL // max(w, 1))          # Alg. 3 line 9 (R12)
            cur_off = len(slot_col)
            if coo and not (split_long_rows and w > WL):
                # whole rows while the workload holds at most WL entries (at least one row), back
                # to back, the last entry of each row flagged (bit 31 of the column), padded to 32
                h, tot = 0, 0
                while i + h < len(rows) and (h == 0 or tot + lens[i + h] <= WL):
                    tot += lens[i + h]
                    h += 1
                wp = _roundup(tot, 32)
                emit(cur_off, len(row_id), wp, h, KIND_COO, 1, -1, 0)
                for r in rows[i:i + h]:
                    row_id.append(flags_for(t, r))
                    ents = per_tile[t][r]
                    for k, (c_, v_) in enumerate(ents):
                        word = c_ | (COO_END if k + 1 == len(ents) else 0)
                        slot_col.append(word - (1 << 32) if word >= (1 << 31) else word)   # as int32
                        if not pattern:
                            slot_val.append(v_)
                for _ in range(wp - tot):
                    slot_col.append(sentinel)
                    if not pattern:
                        slot_val.append(np.float32(0))
                camp()
                i += h
                continue
            if split_long_rows and w > WL:        # R21: one-row chunks of <= WL entries
                r = rows[i]
                ents = per_tile[t][r]
                nch = (w + WL - 1) // WL
                sid = len(split)
                pbase = int(sum(s[1] for s in split))
                split.append((flags_for(t, r), nch, pbase))
                for ch in range(nch):
                    cur_off = len(slot_col)
                    part = ents[ch * WL: min((ch + 1) * WL, w)]
                    wp = _roundup(len(part), align_rm)
                    emit(cur_off, len(row_id), wp, 1, KIND_SPLIT, 4, sid, ch)
                    row_id.append(flags_for(t, r))
                    for k in range(wp):
                        if k < len(part):
                            slot_col.append(part[k][0])
                            if not pattern:
                                slot_val.append(part[k][1])
                        else:
                            slot_col.append(sentinel)
                            if not pattern:
                                slot_val.append(np.float32(0))
                    camp()
                i += 1
                continue
            # Alg. 3's rule (row major iff w >= h); orient 1 / 2 force one format for the
            # single-format special cases the model covers, zero-length rows excepted
            if (w > 0) if orient_t == 1 else (False if orient_t == 2 else w >= hq):   # row major
                h = min(hq, len(rows) - i)
                wp = _roundup(w, align_rm)
                emit(cur_off, len(row_id), wp, h, KIND_RM, 4, -1, 0)
                for r in rows[i:i + h]:
                    row_id.append(flags_for(t, r))
                    ents = per_tile[t].get(r, [])
                    for k in range(wp):
                        if k < len(ents):
                            slot_col.append(ents[k][0])
                            if not pattern:
                                slot_val.append(ents[k][1])
                        else:
                            slot_col.append(sentinel)
                            if not pattern:
                                slot_val.append(np.float32(0))
                i += h
            else:                                  # column major, ELL style
                hp = _roundup(hq, ell_h)
                take = min(hp, len(rows) - i)
                slabs = (take + ell_h - 1) // ell_h
                kvec = 4 if w % 4 == 0 else (2 if w % 2 == 0 else 1)
                emit(cur_off, len(row_id), w, slabs * ell_h, KIND_CM, kvec, -1, 0)
                slab_rows = rows[i:i + take] + [None] * (slabs * ell_h - take)
                for r in slab_rows:
                    row_id.append(PAD_ROW if r is None else flags_for(t, r))
                for s in range(slabs):
                    block_c = [sentinel] * (ell_h * w)
                    block_v = [np.float32(0)] * (ell_h * w)
                    for rr in range(ell_h):
                        r = slab_rows[s * ell_h + rr]
                        ents = [] if r is None else per_tile[t].get(r, [])
                        for k, (c_, v_) in enumerate(ents):
                            pos = (k // kvec) * ell_h * kvec + rr * kvec + (k % kvec)
                            block_c[pos] = c_
                            block_v[pos] = v_
                    slot_col.extend(block_c)
                    if not pattern:
                        slot_val.extend(block_v)
                i += take
            camp()
        tiles[t, 3] = len(desc["off"])

    d = {
        "off": np.array(desc["off"], dtype=np.int64),
        "row_base": np.array(desc["row_base"], dtype=np.int32),
        "w": np.array(desc["w"], dtype=np.int32),
        "h": np.array(desc["h"], dtype=np.int32),
        "kind": np.array(desc["kind"], dtype=np.uint8),
        "kvec": np.array(desc["kvec"], dtype=np.uint8),
        "split_id": np.array(desc["split_id"], dtype=np.int32),
        "chunk": np.array(desc["chunk"], dtype=np.int32),
    }
    return Layout(
        n_rows=n_rows, n_cols=n_cols, pattern=pattern, perm=perm, inv=inv, tiles=tiles, desc=d,
        row_id=np.array(row_id, dtype=np.uint32),
        slot_col=np.array(slot_col, dtype=np.int32),
        slot_val=None if pattern else np.array(slot_val, dtype=np.float32),
        split=np.array(split, dtype=np.int32).reshape(-1, 3),
        meta=dict(tile_width=tile_width, num_tiles=T, workload_sizes=list(workload_sizes),
                  align_rm=align_rm, split=split_long_rows, camping=camping_pad, ell_h=ell_h,
                  collen=collen),
    )


def decode_to_coo(L: Layout):
    """Walk the layout and return the stored (row, original col, value) entries, padding dropped.
    The round-trip property: this multiset equals the input matrix's entries."""
    rows, cols, vals = [], [], []
    n_wl = len(L.desc["off"])
    tile_of_wl = np.zeros(n_wl, dtype=np.int64)
    for t in range(L.tiles.shape[0]):
        tile_of_wl[L.tiles[t, 2]:L.tiles[t, 3]] = t
    ell_h = L.meta["ell_h"]
    for j in range(n_wl):
        t = tile_of_wl[j]
        lo, hi = int(L.tiles[t, 0]), int(L.tiles[t, 1])
        sent = hi - lo
        off, rb, w, h = int(L.desc["off"][j]), int(L.desc["row_base"][j]), int(L.desc["w"][j]), int(L.desc["h"][j])
        kind, kvec = int(L.desc["kind"][j]), int(L.desc["kvec"][j])

        def put(r_entry, s):
            c = int(L.slot_col[s]) & (COO_END - 1)
            if c == sent:
                return
            rows.append(int(r_entry) & (FLAG_ACC - 1))
            cols.append(int(L.perm[lo + c]))
            vals.append(1.0 if L.pattern else float(L.slot_val[s]))
        if kind == KIND_COO:
            r = 0
            for k in range(w):
                if r >= h:
                    break
                put(L.row_id[rb + r], off + k)
                if int(L.slot_col[off + k]) < 0:          # bit 31: the row's last entry
                    r += 1
        elif kind in (KIND_RM, KIND_SPLIT):
            for r in range(h):
                for k in range(w):
                    put(L.row_id[rb + r], off + r * w + k)
        else:
            for r in range(h):
                if L.row_id[rb + r] == PAD_ROW:
                    continue
                s0 = off + (r // ell_h) * ell_h * w
                rr = r % ell_h
                for k in range(w):
                    put(L.row_id[rb + r], s0 + (k // kvec) * ell_h * kvec + rr * kvec + (k % kvec))
    return np.array(rows, dtype=np.int64), np.array(cols, dtype=np.int64), np.array(vals, dtype=np.float64)
