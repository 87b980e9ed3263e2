"""Selector oracle: the history-based variant-selection algorithm, step by step.

TEST INFRASTRUCTURE ONLY — see oracle/__init__.py.  Shares no code with the
C++ runtime (paper_2311_03543_b200/csrc/runtime/selector.cpp); tests drive both
with the same task stream and require identical decisions.

Selection is a heuristic, so this oracle is the algorithm itself, written in the
order of SURVEY.md §8(c) "Selector oracle" steps 1-7, which restate:
  * PAPER.md P:118 [§2.2.2] — "When a task is executed, a codelet is selected
    based on the specific architecture and data associated with it";
  * PAPER.md P:224 [§3.2] — selection by trained performance models,
    "additional training ... could lead to more accurate ... selection";
  * SPEC.md S:363-371 (calibration while < K samples, then argmin of the
    recorded mean), S:376 (every execution records its duration), S:412 (K=3),
    S:416 (ties -> lowest variant index).
Readings that deviate from SPEC on purpose are listed in DESIGN.md (R9-R13):
integer-ns sums instead of Welford, key = (m_panel, n, k, dtype, compute,
transB, beta==0), W=1 warm-up execution per (variant, key) discarded.

Parity pins (tests/test_selector_oracle.py): S:369 alternation (2 variants, K=3
-> 6 alternating runs), S:370-371 closed-form crossover (n=256 -> v0,
n=4096 -> v1), tie -> lowest index, permutation invariance, save/load replay.
"""
from __future__ import annotations

from dataclasses import dataclass, field

# precision classes / targets (mirror include/compar.h values; restated, not imported)
TGT_SIMT_F32, TGT_TMA_F32, TGT_TC_TF32, TGT_TC_BF16, TGT_USER = 0, 1, 2, 3, 4
F32, BF16 = 0, 1
COMPUTE_F32_STRICT, COMPUTE_TF32, COMPUTE_BF16 = 0, 1, 2
MODE_WARMUP, MODE_CALIB, MODE_MODEL, MODE_EAGER, MODE_HINT, MODE_NOOP = 0, 1, 2, 3, 4, 5


def admits(target: int, in_dtype: int, compute: int) -> bool:
    """§8(b) eligibility by precision class (step 1, first half)."""
    if target == TGT_USER:
        return True
    if compute == COMPUTE_BF16:
        return in_dtype == BF16 and target == TGT_TC_BF16
    if in_dtype != F32:
        return False
    if compute == COMPUTE_F32_STRICT:
        return target in (TGT_SIMT_F32, TGT_TMA_F32)
    if compute == COMPUTE_TF32:
        return target in (TGT_SIMT_F32, TGT_TMA_F32, TGT_TC_TF32)
    return False


def tma_ok(elem_bytes: int, ptrs, lds) -> bool:
    """TMA constraint (step 1, second half): 16-B aligned bases, ld*elem % 16 == 0."""
    return all(p % 16 == 0 for p in ptrs) and all((ld * elem_bytes) % 16 == 0 for ld in lds)


@dataclass
class Record:
    seen: int = 0          # executions assigned (warm-up + timed + pending)
    count: int = 0         # timed samples harvested
    sum_ns: int = 0
    sumsq_ns: int = 0
    min_ns: int = 0


@dataclass
class SelectorOracle:
    n_variants: int
    calib_warmup: int = 1      # W
    calib_k: int = 3           # K_cal
    eager: bool = False
    hist: dict = field(default_factory=dict)   # (v, key) -> Record

    def rec(self, v: int, key) -> Record:
        return self.hist.setdefault((v, key), Record())

    def decide(self, key, eligible):
        """Steps 3-5 and 7: return (variant, mode) for the next execution of `key`.

        `eligible` is the ordered list E of eligible variant indices (step 1).
        Assumes all pending samples have been harvested when model mode is
        reached (step 6 is the caller's blocking harvest)."""
        if not eligible:
            raise LookupError("E_NO_VARIANT")
        if self.eager:
            return eligible[0], MODE_EAGER
        need = self.calib_warmup + self.calib_k
        seen = [self.rec(v, key).seen for v in eligible]
        if min(seen) < need:                                   # step 4: calibration
            best = min(range(len(eligible)), key=lambda t: (seen[t], eligible[t]))
            v = eligible[best]
            return v, (MODE_WARMUP if seen[best] < self.calib_warmup else MODE_CALIB)
        best_v = None                                           # step 5: model
        for v in eligible:
            r = self.rec(v, key)
            if r.count == 0:
                continue
            if best_v is None:
                best_v = v
                continue
            b = self.rec(best_v, key)
            # mean(v) < mean(best) <=> sum_v * count_b < sum_b * count_v (exact integers)
            if r.sum_ns * b.count < b.sum_ns * r.count:
                best_v = v
        if best_v is None:
            best_v = eligible[0]
        return best_v, MODE_MODEL

    def commit(self, v: int, key, mode: int) -> bool:
        """Account a submitted execution; returns True if it is a warm-up."""
        if mode in (MODE_EAGER, MODE_HINT, MODE_NOOP):
            return False
        r = self.rec(v, key)
        warm = r.seen < self.calib_warmup
        r.seen += 1
        return warm

    def harvest(self, v: int, key, mode: int, warm: bool, ns: int) -> None:
        """Step 7 / a9: append a timed sample (integer ns); warm-ups are dropped."""
        if mode in (MODE_EAGER, MODE_HINT, MODE_NOOP) or warm:
            return
        r = self.rec(v, key)
        r.min_ns = ns if r.count == 0 else min(r.min_ns, ns)
        r.count += 1
        r.sum_ns += ns
        r.sumsq_ns += ns * ns

    def mean_ns(self, v: int, key) -> float:
        r = self.rec(v, key)
        return r.sum_ns / r.count if r.count else float("inf")
