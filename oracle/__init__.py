"""COMPAR oracle — plain, slow, obviously-correct CPU reference.  TEST INFRASTRUCTURE.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline /
`--impl reference` legs may import, call, link or execute anything here.  The
product path (`paper_2311_03543_b200/`, `include/compar.h`) never does, and this
package imports nothing from it.  The two sides share only the seeded input
generator package `gen/`, which contains no GEMM arithmetic.

Contents and what pins each one (DESIGN.md §4 lists the same table):

* `gemm.py` + `gemm_oracle.c` — FP64 triple-loop GEMM, PAPER.md P:76-80 and
  P:201-205 read as xGEMM (C = alpha*A*B + beta*C).  Pinned by worked examples
  (tests/golden/gemm_*.txt), closed forms (identity, diagonal, rank-1, ones),
  exact-rational brute force and numpy float64 cross-checks.
* `selector.py` — history selector steps 1-7 (SPEC S:363-371,
  S:412).  Pinned by the S:369 alternation, the S:370-371 closed-form
  crossover and tie/permutation invariants.
* `partition.py` — row-panel formula (north star; reading R14).  Pinned by
  coverage/disjointness/alignment invariants and hand-computed cases.

Selection QUALITY (which variant is fastest on B200) is hardware-dependent:
"parity unpinned" — only regret against exhaustive
measurement is checkable, and bench/selector reports it.
"""
