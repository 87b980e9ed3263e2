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

import math
from dataclasses import dataclass, field

# precision classes / targets (mirror include/compar.h values; restated, not imported)
TGT_SIMT_F32, TGT_TMA_F32, TGT_TC_TF32, TGT_TC_BF16, TGT_USER = 0, 1, 2, 3, 4
TGT_SIMT_BF16 = 9
TGT_TCX_F32 = 14
F32, BF16 = 0, 1
COMPUTE_F32_STRICT, COMPUTE_TF32, COMPUTE_BF16, COMPUTE_F32_SPLIT = 0, 1, 2, 3
MODE_WARMUP, MODE_CALIB, MODE_MODEL, MODE_EAGER, MODE_HINT, MODE_NOOP, MODE_PREDICT = 0, 1, 2, 3, 4, 5, 6


def admits(target: int, in_dtype: int, compute: int) -> bool:
    """§8(b) eligibility by precision class (step 1, first half)."""
    if target == TGT_USER:
        return True
    if compute == COMPUTE_BF16:
        return in_dtype == BF16 and target in (TGT_TC_BF16, TGT_SIMT_BF16)
    if in_dtype != F32:
        return False
    if compute == COMPUTE_F32_STRICT:
        return target in (TGT_SIMT_F32, TGT_TMA_F32)
    if compute == COMPUTE_TF32:
        return target in (TGT_SIMT_F32, TGT_TMA_F32, TGT_TC_TF32)
    if compute == COMPUTE_F32_SPLIT:   # FP32 accuracy: the FFMA variants and the split TF32 form (R38)
        return target in (TGT_SIMT_F32, TGT_TMA_F32, TGT_TCX_F32)
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
    blocked: bool = False      # calibration order (R19); False = SPEC S:369 interleaving
    explore_pct: int = 150     # DESIGN.md R37 predict-mode exploration threshold (percent)
    long_warm_ms: int = 200    # DESIGN.md R39: warm-up time for variants whose lower bound is >= 10 ms
    prune_pct: int = 150       # DESIGN.md R32 calibration pruning threshold (percent, the runtime default); 0 = SPEC
    hist: dict = field(default_factory=dict)   # (v, key) -> Record

    def rec(self, v: int, key) -> Record:
        return self.hist.setdefault((v, key), Record())

    # ---- R32: calibration pruning.  Written from the rule: let best = the smallest measured mean
    # over the eligible variants of the key; a variant is done calibrating once its own mean, or its
    # static lower bound lb (ns), exceeds prune_pct / 100 x best.
    def best_mean(self, key, eligible):
        """(sum, count) of the smallest mean, or None if no eligible variant has a sample."""
        best = None
        for v in eligible:
            r = self.rec(v, key)
            if r.count and (best is None or r.sum_ns * best[1] < best[0] * r.count):
                best = (r.sum_ns, r.count)
        return best

    def pruned(self, key, eligible, t, lb=None):
        if self.prune_pct <= 0:
            return False
        best = self.best_mean(key, eligible)
        if best is None:
            return False
        bs, bc = best
        r = self.rec(eligible[t], key)
        if r.count and 100 * r.sum_ns * bc > self.prune_pct * bs * r.count:
            return True
        lv = lb[t] if lb else 0.0
        return lv > 0.0 and lv * 100.0 * float(bc) > float(self.prune_pct) * float(bs)

    def warm_count(self, lb_ns=0.0):
        """R39, written from the rule: a variant whose static lower bound is at least 10 ms gets
        ceil(long_warm_ms / lb) warm-up executions (at least W, at most 6) — enough to run ~200 ms
        before its timed samples; every other variant gets W."""
        if self.long_warm_ms <= 0 or lb_ns < 10e6:
            return self.calib_warmup
        w = math.ceil(self.long_warm_ms * 1e6 / lb_ns)
        return min(6, max(self.calib_warmup, w))

    def calibrating(self, key, eligible, lb=None):
        return any(self.rec(v, key).seen < self.warm_count(lb[t] if lb else 0.0) + self.calib_k
                   and not self.pruned(key, eligible, t, lb)
                   for t, v in enumerate(eligible))

    def decide(self, key, eligible, lb=None):
        """Steps 3-5 and 7: return (variant, mode) for the next execution of `key`.

        `eligible` is the ordered list E of eligible variant indices (step 1); `lb` the static
        lower bounds (ns) in the same order (R32), None = none.  Assumes all pending samples have
        been harvested when model mode is reached (step 6 is the caller's blocking harvest)."""
        if not eligible:
            raise LookupError("E_NO_VARIANT")
        if self.eager:
            return eligible[0], MODE_EAGER
        warm = [self.warm_count(lb[t] if lb else 0.0) for t in range(len(eligible))]
        seen = [self.rec(v, key).seen for v in eligible]
        cand = [t for t in range(len(eligible))
                if seen[t] < warm[t] + self.calib_k and not self.pruned(key, eligible, t, lb)]
        if cand:                                               # step 4: calibration
            if self.blocked:   # R19 / R32: finish one variant's W + K executions before the next,
                # visiting variants by increasing lower bound (ties: eligibility order)
                best = min(cand, key=lambda t: ((lb[t] if lb else 0.0), t))
            else:
                best = min(cand, key=lambda t: (seen[t], eligible[t]))
            v = eligible[best]
            return v, (MODE_WARMUP if seen[best] < warm[best] else MODE_CALIB)
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

    def commit(self, v: int, key, mode: int, lb_ns: float = 0.0) -> bool:
        """Account a submitted execution (lb_ns: the variant's static lower bound, R39); returns
        True if it is a warm-up."""
        if mode in (MODE_EAGER, MODE_HINT, MODE_NOOP):  # MODE_PREDICT executions are accounted
            return False
        r = self.rec(v, key)
        warm = r.seen < self.warm_count(lb_ns)
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

    # ---- NEXT-2 "predict" scheduler (PAPER.md P:224 / P:308 "additional training").
    # key = (m, n, k, dtype, compute, transB, beta0).  Written from the definition: weighted least
    # squares with weights 1/t^2 over every non-empty subset of the features {1, GFLOP, MB},
    # keep the non-negative solution of least relative residual.
    MIN_FIT_KEYS = 3

    @staticmethod
    def features(key):
        m, n, k, dtype, _compute, _tb, beta0 = key
        eb = 2.0 if dtype == BF16 else 4.0
        return [1.0, 2.0 * m * n * k * 1e-9, (eb * (m * k + k * n) + 4.0 * m * n * (1.0 if beta0 else 2.0)) * 1e-6]

    def predict(self, v: int, key):
        import numpy as np
        pts = [(self.features(kk), r.sum_ns / r.count) for (vv, kk), r in self.hist.items()
               if vv == v and r.count > 0 and kk[3:6] == key[3:6]]
        if len(pts) < self.MIN_FIT_KEYS:
            return None
        X = np.array([p[0] for p in pts])
        t = np.array([p[1] for p in pts])
        wt = 1.0 / (t * t + 1.0)
        best = None
        for mask in range(1, 8):
            cols = [j for j in range(3) if mask >> j & 1]
            Xs = X[:, cols]
            a = (Xs * wt[:, None]).T @ Xs
            b = (Xs * wt[:, None]).T @ t
            try:
                w = np.linalg.solve(a, b)
            except np.linalg.LinAlgError:
                continue
            if (w < 0).any():
                continue
            full = np.zeros(3)
            full[cols] = w
            res = float((((X @ full) - t) / t) ** 2 @ np.ones(len(t)))
            if best is None or res < best[0]:
                best = (res, full)
        if best is None:
            return None
        return float(np.array(self.features(key)) @ best[1])

    def _estimates(self, key, eligible):
        """Per eligible variant: (estimate ns, predicted?) or None — measured mean, else the fit."""
        out = []
        for v in eligible:
            r = self.rec(v, key)
            if r.count > 0:
                out.append((r.sum_ns / r.count, False))
            else:
                p = self.predict(v, key)
                out.append(None if p is None else (p, True))
        return out

    def _lb_skipped(self, est, t, lb):
        """R32 in predict mode: a variant with no estimate whose lower bound exceeds prune_pct/100
        x the best known estimate is not calibrated."""
        known = [e[0] for e in est if e is not None]
        lv = lb[t] if lb else 0.0
        return bool(known) and self.prune_pct > 0 and lv > 0.0 and lv * 100.0 > float(self.prune_pct) * min(known)

    def unknown_predict(self, key, eligible, lb=None):
        """Variants with neither samples for `key` nor a fitted prediction (nor skipped by their
        lower bound); in predict mode only these are calibrated when decide_predict returns None."""
        est = self._estimates(key, eligible)
        return [v for t, v in enumerate(eligible) if est[t] is None and not self._lb_skipped(est, t, lb)]

    def decide_predict(self, key, eligible, lb=None):
        """Measured mean where (v, key) has samples, else the fitted prediction; None if some
        eligible variant has neither (the caller then calibrates) and is not skipped by R32."""
        est = self._estimates(key, eligible)
        best = None
        for t, v in enumerate(eligible):
            if est[t] is None:
                if self._lb_skipped(est, t, lb):
                    continue
                return None
            if best is None or est[t][0] < best[1]:
                best = (v, est[t][0], est[t][1])
        if best is None:
            return None
        if not best[2] and self.explore_pct > 0:
            # R37: the best estimate is a measured mean; a variant known only by its prediction,
            # predicted within explore_pct/100 of it, is measured (W + 1 runs) before it is trusted
            for t, v in enumerate(eligible):
                if est[t] is not None and est[t][1] and est[t][0] * 100.0 <= float(self.explore_pct) * best[1]:
                    return v, (MODE_WARMUP if self.rec(v, key).seen < self.warm_count(lb[t] if lb else 0.0)
                               else MODE_CALIB)
        return best[0], (MODE_PREDICT if best[2] else MODE_MODEL)

    # ---- R32 static lower bound of a built-in GEMM variant (mirrors the runtime's class peaks,
    # restated): FLOPs at the nominal peak of its class, compulsory bytes at nominal 8 TB/s.
    @staticmethod
    def static_lb_ns(cls, key, sms=148):
        """cls: 'ffma' | 'bf16' | 'tf32' | 'f32x3' | None (USER: no bound).  'f32x3' (R38) runs three
        TF32 products per FP32 product: a third of the TF32 peak."""
        if cls is None:
            return 0.0
        peak = {"ffma": float(sms) * 128.0 * 2.0 * 1.965e9, "bf16": 2.25e15, "tf32": 1.125e15,
                "f32x3": 1.125e15 / 3.0}[cls]
        m, n, k, dtype, _c, _t, beta0 = key
        m, n, k = float(m), float(n), float(k)
        flops = 2.0 * m * n * k
        eb = 2.0 if dtype == BF16 else 4.0
        nbytes = eb * (m * k + k * n) + 4.0 * m * n * (1.0 if beta0 else 2.0)
        return max(flops / peak, nbytes / 8.0e12) * 1e9
