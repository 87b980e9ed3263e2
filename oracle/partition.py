"""Row-panel partition oracle.  TEST INFRASTRUCTURE ONLY.

The paper runs on one GPU (PAPER.md P:153 [Table 1]) and leaves "mapping,
scheduling" to the runtime (P:118 [§2.2.2]); the multi-GPU row-panel split is
the north star's (BASELINE.json).  Reading R14: panels are aligned
to the 128-row tensor-core tile:

    base = ceil(ceil(M / P) / 128) * 128 ;  o_r = min(M, r * base) ;  o_P = M

panel r = rows [o_r, o_{r+1}) of A and C; empty panels are skipped.  Because no
split-K is used, C is the row-concatenation of the panel products:
C[o_r:o_{r+1}] = alpha * A[o_r:o_{r+1}] @ B + beta * C_in[o_r:o_{r+1}].
"""
from __future__ import annotations


def partition_rows(m: int, p: int, align: int = 128) -> list[int]:
    if m < 0 or p < 1:
        raise ValueError("bad partition arguments")
    per = -(-m // p)
    base = -(-per // align) * align
    offs = [min(m, r * base) for r in range(p)]
    offs.append(m)
    return offs
