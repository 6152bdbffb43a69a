"""partition_ref -- TEST INFRASTRUCTURE ONLY.  Bitonic (snake) row partition of Sec. 3.2.

PAPER.md L108: "The matrix rows are first sorted by length. Each iteration of the algorithm
processes P rows and assigns them to P processors. The processor that got the longest row in the
previous iteration will get the shortest row in the current iteration."
Reading R25/O6: rows ordered by (length desc, id asc); sorted position s goes to rank s mod P
when floor(s/P) is even, else to P-1-(s mod P).  The final partial group follows the same rule.
"""
from __future__ import annotations


def bitonic_partition(row_len, P: int):
    """Returns owner[i] for every row i (plain Python, one row at a time)."""
    n = len(row_len)
    if P < 1 or P > max(n, 1):
        raise ValueError("P must satisfy 1 <= P <= rows")
    order = sorted(range(n), key=lambda i: (-int(row_len[i]), i))
    owner = [0] * n
    for s, i in enumerate(order):
        g, j = divmod(s, P)
        owner[i] = j if g % 2 == 0 else P - 1 - j
    return owner
