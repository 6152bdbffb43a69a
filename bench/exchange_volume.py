"""Per-iteration exchange volume of the row-partitioned PageRank, host only.

For the bitonic row partition of the iteration matrix M = A^T over P ranks, floats received per
iteration summed over all ranks, for three exchanges:
  allgather   -- every rank receives every other rank's slot of non-empty columns (the default
                 path: P-1 slots of S_ex floats each, S_ex = the largest per-rank count);
  needed      -- each rank receives only the values its rows read (exchange = 1, spmv_needed_lists);
  column      -- the column partition the paper compares against: each rank owns the
                 same vertices as columns, produces partial y for every row its columns touch, and
                 sends the partials of rows it does not own (= the needed volume of M^T);
  grid        -- the 2-D (grid) partition: ranks form pr x pc (pr <= pc), vertex v's
                 owner r(v) gives its row group r // pc and column group r % pc; rank (i, j) holds
                 the entries of rows in group i and columns in group j, receives the x values of
                 its columns it does not own and sends the partial y of its rows it does not own
                 (x broadcast within the column group + partial-y reduction within the row group).
Usage: python bench/exchange_volume.py c2 [c4 ...] > profiles/r02_exchange_volume.jsonl"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import graphgen  # noqa: E402
from paper_1103_2405_b200 import needed_lists, partition_plan  # noqa: E402


def grid_volume(rp, col, owner, P):
    """floats received per iteration, summed over ranks, by the pr x pc grid partition"""
    pr = int(np.floor(np.sqrt(P)))
    while P % pr:
        pr -= 1
    pc = P // pr
    n = len(rp) - 1
    v = np.repeat(np.arange(n, dtype=np.int64), np.diff(rp))          # row of each entry
    u = col.astype(np.int64)                                           # column of each entry
    ov, ou = owner[v].astype(np.int64), owner[u].astype(np.int64)
    h = (ov // pc) * pc + (ou % pc)                                    # holder rank of the entry
    xk = np.unique(h * n + u)                                          # (holder, column) pairs
    x_in = int(np.count_nonzero(owner[xk % n] != xk // n))
    yk = np.unique(h * n + v)                                          # (holder, row) pairs
    y_out = int(np.count_nonzero(owner[yk % n] != yk // n))
    return x_in + y_out, f"{pr}x{pc}"


def main():
    for cfg in sys.argv[1:] or ["c2"]:
        t0 = time.time()
        G = graphgen.make_graph(cfg)
        n = G.n
        outdeg = np.diff(G.row_ptr)
        rp, col = graphgen.keys_to_csr(G.keys, n, transpose=True)      # M = A^T: row v reads u -> v
        for P in (2, 4, 8):
            owner, _, _ = partition_plan(np.diff(rp), P)
            ne = outdeg > 0
            s_ex = int(np.bincount(owner[ne], minlength=P).max())
            allgather = P * (P - 1) * s_ex
            needed = sum(int(sum(len(v) for v in needed_lists(rp, col, owner, P, r)[1])) for r in range(P))
            column = sum(int(sum(len(v) for v in needed_lists(G.row_ptr, G.col, owner, P, r)[1])) for r in range(P))
            grid, shape = grid_volume(rp, col, owner, P)
            print(json.dumps(dict(config=cfg, n=n, m=int(len(col)), P=P, dangling_frac=round(float((~ne).mean()), 4),
                                  allgather_floats=allgather, needed_floats=needed, column_floats=column,
                                  needed_vs_allgather=round(needed / max(allgather, 1), 4),
                                  column_vs_allgather=round(column / max(allgather, 1), 4),
                                  grid_shape=shape, grid_floats=grid,
                                  grid_vs_allgather=round(grid / max(allgather, 1), 4),
                                  elapsed_s=round(time.time() - t0, 1))), flush=True)


if __name__ == "__main__":
    main()
