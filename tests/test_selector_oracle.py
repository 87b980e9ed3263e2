"""Pins of the selector and partition oracles (oracle/selector.py, oracle/partition.py)."""
import itertools
import random

import pytest

from oracle import selector as so
from oracle.partition import partition_rows


def run_stream(sel, key, eligible, cost, n_runs):
    """Drive the oracle with synthetic costs (virtual clock): returns the (v, mode) trace."""
    trace = []
    for _ in range(n_runs):
        v, mode = sel.decide(key, eligible)
        warm = sel.commit(v, key, mode)
        sel.harvest(v, key, mode, warm, cost(v))
        trace.append((v, mode))
    return trace


def test_spec_s369_alternation():
    """2 variants, unseen key, K=3 -> the first 6 executions alternate (3 each)."""
    sel = so.SelectorOracle(2, calib_warmup=0, calib_k=3)
    trace = run_stream(sel, "k", [0, 1], lambda v: 100 + v, 6)
    assert [v for v, _ in trace] == [0, 1, 0, 1, 0, 1]
    assert all(m == so.MODE_CALIB for _, m in trace)
    v, m = sel.decide("k", [0, 1])
    assert m == so.MODE_MODEL and v == 0


def test_config1_calibration_plan():
    """3 variants x (1 warm-up + 3 timed) = 12 calibration runs in order 0,1,2,... then model
    (the SPEC S:369 plan: calibration pruning off, R32)."""
    sel = so.SelectorOracle(3, prune_pct=0)
    trace = run_stream(sel, "k", [0, 1, 2], lambda v: [30, 10, 20][v], 13)
    assert [v for v, _ in trace[:12]] == [0, 1, 2] * 4
    assert [m for _, m in trace[:3]] == [so.MODE_WARMUP] * 3
    assert all(m == so.MODE_CALIB for _, m in trace[3:12])
    assert trace[12] == (1, so.MODE_MODEL)


def test_blocked_calibration_plan():
    """R19 blocked order: W + K executions of each variant back to back, in eligibility order."""
    sel = so.SelectorOracle(3, blocked=True)
    trace = run_stream(sel, "k", [2, 0, 1], lambda v: [30, 10, 20][v], 13)
    assert [v for v, _ in trace[:12]] == [2] * 4 + [0] * 4 + [1] * 4
    assert [m for _, m in trace[:12]] == ([so.MODE_WARMUP] + [so.MODE_CALIB] * 3) * 3
    assert trace[12] == (1, so.MODE_MODEL)
    # a variant that becomes eligible later is calibrated next, as a block
    trace = run_stream(sel, "k", [2, 0, 1, 3], lambda v: [30, 10, 20, 5][v], 5)
    assert [v for v, _ in trace] == [3, 3, 3, 3, 3] and trace[-1][1] == so.MODE_MODEL


def test_spec_s370_closed_form_crossover(golden):
    """cost0 = 0.1n, cost1 = 50 + 0.01n -> n=256 -> 0, n=4096 -> 1."""
    g = golden("selector_crossover.txt")
    expect = {256: 0, 4096: 1}
    for n, want in expect.items():
        sel = so.SelectorOracle(2)
        costs = [round(0.1 * n * 1000), round((50 + 0.01 * n) * 1000)]   # ns
        run_stream(sel, ("n", n), [0, 1], lambda v: costs[v], 8)
        assert sel.decide(("n", n), [0, 1]) == (want, so.MODE_MODEL)
    assert float(g["crossover"]) == pytest.approx(50 / 0.09)


def test_omniscient_accuracy_is_one():
    """a truthful model picks the argmin at every size (accuracy 1.0)."""
    sel = so.SelectorOracle(2)
    for n in [64, 128, 256, 512, 555, 556, 600, 1024, 4096]:
        c = [round(100 * n), round(50000 + 10 * n)]
        run_stream(sel, n, [0, 1], lambda v: c[v], 8)
        v, _ = sel.decide(n, [0, 1])
        assert v == min((0, 1), key=lambda t: (c[t], t))


def test_tie_goes_to_lowest_index_and_eligibility_order():
    sel = so.SelectorOracle(3)
    run_stream(sel, "k", [0, 1, 2], lambda v: 500, 12)
    assert sel.decide("k", [0, 1, 2]) == (0, so.MODE_MODEL)
    assert sel.decide("k", [1, 2]) == (1, so.MODE_MODEL)


def test_permutation_invariance_of_samples():
    """Integer sums: harvest order does not change the model decision (exact here)."""
    samples = [(0, 1003), (0, 997), (0, 1000), (1, 999), (1, 1001), (1, 1000)]
    decisions = set()
    for perm in itertools.permutations(samples):
        sel = so.SelectorOracle(2, calib_warmup=0)
        for v, _ in [(0, 0), (1, 0)] * 3:
            sel.commit(v, "k", so.MODE_CALIB)
        for v, ns in perm:
            sel.harvest(v, "k", so.MODE_CALIB, False, ns)
        decisions.add(sel.decide("k", [0, 1]))
    assert decisions == {(0, so.MODE_MODEL)}          # exact tie 3000 vs 3000 -> index 0


def test_eager_and_no_variant():
    sel = so.SelectorOracle(3, eager=True)
    assert sel.decide("k", [2, 1]) == (2, so.MODE_EAGER)
    with pytest.raises(LookupError):
        sel.decide("k", [])


def test_admits_table():
    """§8(b) eligibility: strict FP32 -> SIMT, TMA; TF32 -> + TC_TF32; BF16 -> TC_BF16 only."""
    f32, bf16 = so.F32, so.BF16
    el = lambda d, c: [t for t in range(4) if so.admits(t, d, c)]
    assert el(f32, so.COMPUTE_F32_STRICT) == [0, 1]
    assert el(f32, so.COMPUTE_TF32) == [0, 1, 2]
    assert el(bf16, so.COMPUTE_BF16) == [3]
    assert so.admits(so.TGT_SIMT_BF16, bf16, so.COMPUTE_BF16) and not so.admits(so.TGT_SIMT_BF16, f32, so.COMPUTE_TF32)
    assert el(bf16, so.COMPUTE_TF32) == []
    # F32_SPLIT (R38): FP32 accuracy -> the FFMA variants and the TF32-split form, never plain TF32
    assert el(f32, so.COMPUTE_F32_SPLIT) == [0, 1]
    assert so.admits(so.TGT_TCX_F32, f32, so.COMPUTE_F32_SPLIT)
    assert not any(so.admits(so.TGT_TCX_F32, f32, c) for c in (so.COMPUTE_F32_STRICT, so.COMPUTE_TF32))
    assert not so.admits(so.TGT_TCX_F32, bf16, so.COMPUTE_F32_SPLIT)
    assert so.tma_ok(4, [0, 256], [64, 8]) and not so.tma_ok(4, [4], [64]) and not so.tma_ok(2, [0], [9])


def _key(s, beta0=0):
    return (s, s, s, so.F32, so.COMPUTE_TF32, 0, beta0)


def test_predict_recovers_closed_form():
    """NEXT-2 pin: with exact affine costs t = a + b * GFLOP the weighted fit recovers them, so the
    prediction at an unseen size equals the closed form and the decision is its argmin."""
    sel = so.SelectorOracle(2)
    cost = [lambda s: 50_000 + 900.0 * 2 * s ** 3 * 1e-9, lambda s: 5_000 + 2_000.0 * 2 * s ** 3 * 1e-9]
    for s in (256, 512, 1024, 2048):
        for _ in range(8):
            v, mode = sel.decide(_key(s), [0, 1])
            warm = sel.commit(v, _key(s), mode)
            sel.harvest(v, _key(s), mode, warm, round(cost[v](s)))
    for s in (3000, 600, 8192):
        for v in (0, 1):
            assert sel.predict(v, _key(s)) == pytest.approx(cost[v](s), rel=1e-3)   # samples are integer ns
        v, mode = sel.decide_predict(_key(s), [0, 1])
        assert mode == so.MODE_PREDICT and v == min((0, 1), key=lambda t: cost[t](s))
    # not enough keys for a variant -> no prediction
    assert so.SelectorOracle(2).decide_predict(_key(64), [0, 1]) is None


def test_predict_calibrates_only_unknown_variants():
    """Predict mode with a variant eligible on too few keys to fit (like the split-K variant): at a
    new key only that variant is calibrated — until its first timed sample, after which (as for every
    variant in predict mode) its measured mean competes with the others' predictions."""
    sel = so.SelectorOracle(3, blocked=True)
    cost = [lambda s: 50_000 + 900.0 * 2 * s ** 3 * 1e-9, lambda s: 5_000 + 2_000.0 * 2 * s ** 3 * 1e-9,
            lambda s: 1_000.0]
    for s in (256, 512, 1024, 2048):                       # variant 2 not eligible on these keys
        for _ in range(8):
            v, mode = sel.decide(_key(s), [0, 1])
            warm = sel.commit(v, _key(s), mode)
            sel.harvest(v, _key(s), mode, warm, round(cost[v](s)))
    key = _key(3000)
    assert sel.decide_predict(key, [0, 1, 2]) is None
    assert sel.unknown_predict(key, [0, 1, 2]) == [2]
    trace = []
    while sel.decide_predict(key, [0, 1, 2]) is None:
        v, mode = sel.decide(key, sel.unknown_predict(key, [0, 1, 2]))
        trace.append((v, mode))
        warm = sel.commit(v, key, mode)
        sel.harvest(v, key, mode, warm, round(cost[v](3000)))
    assert trace == [(2, so.MODE_WARMUP), (2, so.MODE_CALIB)]
    assert sel.decide_predict(key, [0, 1, 2]) == (2, so.MODE_MODEL)   # its measured 1 us beats both predictions


def test_predict_explores_close_predictions():
    """R37 pin: when the best estimate of a key is a measured mean, a variant known only by its
    prediction and predicted within explore_pct/100 of it is measured (one warm-up, one timed run)
    before the measured variant is trusted; one predicted beyond that factor is never run."""
    gf = lambda s: 2 * s ** 3 * 1e-9
    fit = [lambda s: 10_000 + 1000.0 * gf(s), lambda s: 10_000 + 1100.0 * gf(s), lambda s: 10_000 + 2500.0 * gf(s)]

    def trained(explore):
        sel = so.SelectorOracle(3)
        sel.explore_pct = explore
        for s in (256, 512, 1024, 2048):
            for _ in range(12):
                v, mode = sel.decide(_key(s), [0, 1, 2])
                warm = sel.commit(v, _key(s), mode)
                sel.harvest(v, _key(s), mode, warm, round(fit[v](s)))
        return sel

    key = _key(3000)
    actual = [round(fit[0](3000)), 40_000, round(fit[2](3000))]   # variant 1 beats its own prediction here
    for explore, expect in ((150, [(1, so.MODE_WARMUP), (1, so.MODE_CALIB), (1, so.MODE_MODEL)]),
                            (0, [(0, so.MODE_MODEL)] * 3)):
        sel = trained(explore)
        for _ in range(4):                                  # variant 0 measured at the key
            v, mode = sel.decide(key, [0])
            warm = sel.commit(v, key, mode)
            sel.harvest(v, key, mode, warm, actual[v])
        assert sel.predict(1, key) <= 1.5 * actual[0] < sel.predict(2, key)
        trace = []
        for _ in range(3):
            v, mode = sel.decide_predict(key, [0, 1, 2])
            trace.append((v, mode))
            warm = sel.commit(v, key, mode)
            sel.harvest(v, key, mode, warm, actual[v])
        assert trace == expect


@pytest.mark.parametrize("m,p,expect", [
    (32768, 8, [0, 4096, 8192, 12288, 16384, 20480, 24576, 28672, 32768]),
    (32768, 2, [0, 16384, 32768]),
    (1000, 3, [0, 384, 768, 1000]),
    (100, 4, [0, 100, 100, 100, 100]),
    (0, 2, [0, 0, 0]),
    (64, 1, [0, 64]),
])
def test_partition_hand_cases(m, p, expect):
    assert partition_rows(m, p) == expect


def test_partition_invariants():
    rnd = random.Random(1)
    for _ in range(500):
        m, p = rnd.randint(0, 100000), rnd.randint(1, 8)
        o = partition_rows(m, p)
        assert o[0] == 0 and o[-1] == m and len(o) == p + 1
        assert all(a <= b for a, b in zip(o, o[1:]))
        assert all(x % 128 == 0 for x in o[:-1] if x < m)       # panel starts are tile-aligned
        sizes = [b - a for a, b in zip(o, o[1:])]
        assert max(sizes) - min(s for s in sizes if s > 0 or m == 0) <= 128 * p if m else True


# ---- DESIGN.md R32: calibration pruning, hand-derived plans
def test_prune_stops_a_slow_variant_after_one_timed_sample():
    """Blocked, costs 1000 / 5000 / 1100, P = 300 %: v0 calibrates fully (mean 1000); v1's warm-up
    is dropped and its first timed sample (5000 > 3 x 1000) ends its calibration; v2 calibrates
    fully; then model picks v0.  10 executions instead of 12."""
    sel = so.SelectorOracle(3, blocked=True, prune_pct=300)
    trace = run_stream(sel, "k", [0, 1, 2], lambda v: [1000, 5000, 1100][v], 11)
    assert [v for v, _ in trace[:10]] == [0] * 4 + [1] * 2 + [2] * 4
    assert trace[10] == (0, so.MODE_MODEL)
    # without pruning (SPEC behaviour) every variant runs W + K = 4 times
    sel0 = so.SelectorOracle(3, blocked=True, prune_pct=0)
    assert [v for v, _ in run_stream(sel0, "k", [0, 1, 2], lambda v: [1000, 5000, 1100][v], 12)] == \
        [0] * 4 + [1] * 4 + [2] * 4


def test_prune_boundary_is_strict():
    """Exactly 3 x the best mean is NOT pruned (the rule is 'exceeds'); 3 x + 1 ns is."""
    for slow, runs in ((3000, 4), (3001, 2)):
        sel = so.SelectorOracle(2, blocked=True, prune_pct=300)
        trace = run_stream(sel, "k", [0, 1], lambda v: [1000, slow][v], 4 + runs + 1)
        assert [v for v, _ in trace[:4 + runs]] == [0] * 4 + [1] * runs
        assert trace[-1] == (0, so.MODE_MODEL)


def test_prune_static_lower_bound_orders_and_skips():
    """Static lower bounds lb = [3000, 100, 100], costs [10000, 1000, 1000]: blocked calibration
    visits v1, v2 first (smaller lb), then v0 whose lb is exactly 3 x best (not pruned) runs until
    its first timed sample; with lb0 = 3001 v0 never runs at all."""
    key, E = "k", [0, 1, 2]
    cost = lambda v: [10000, 1000, 1000][v]  # noqa: E731
    for lb0, v0_runs in ((3000, 2), (3001, 0)):
        sel = so.SelectorOracle(3, blocked=True, prune_pct=300)
        lb = [float(lb0), 100.0, 100.0]
        trace = []
        for _ in range(8 + v0_runs + 1):
            v, mode = sel.decide(key, E, lb)
            warm = sel.commit(v, key, mode)
            sel.harvest(v, key, mode, warm, cost(v))
            trace.append((v, mode))
        assert [v for v, _ in trace[:8 + v0_runs]] == [1] * 4 + [2] * 4 + [0] * v0_runs
        assert trace[-1] == (1, so.MODE_MODEL)


def test_static_lower_bound_closed_form():
    """lb = max(FLOPs / class peak, bytes / 8 TB/s): 8192^3 BF16 (beta != 0) is compute-bound on
    the tensor cores (2 * 8192^3 / 2.25e15 s = 488.67 us) and on the FFMA pipes of 148 SMs at
    1965 MHz (2 * 8192^3 / 74.45e12 s); 65536 x 256 x 4096 BF16 is bandwidth-bound for the tensor
    class (673.2 MB / 8 TB/s = 84.15 us)."""
    k = (8192, 8192, 8192, so.BF16, so.COMPUTE_BF16, 0, 0)
    assert so.SelectorOracle.static_lb_ns("bf16", k) == pytest.approx(2 * 8192 ** 3 / 2.25e15 * 1e9)
    assert so.SelectorOracle.static_lb_ns("ffma", k) == pytest.approx(2 * 8192 ** 3 / (148 * 256 * 1.965e9) * 1e9)
    assert so.SelectorOracle.static_lb_ns("tf32", (8192, 8192, 8192, so.F32, so.COMPUTE_TF32, 0, 1)) == \
        pytest.approx(2 * 8192 ** 3 / 1.125e15 * 1e9)
    ts = (65536, 256, 4096, so.BF16, so.COMPUTE_BF16, 0, 0)
    nbytes = 2 * (65536 * 4096 + 4096 * 256) + 4 * 65536 * 256 * 2
    assert so.SelectorOracle.static_lb_ns("bf16", ts) == pytest.approx(nbytes / 8e12 * 1e9)
    assert so.SelectorOracle.static_lb_ns(None, ts) == 0.0


def test_long_kernel_warmup_rule():
    """R39 closed forms: W for variants whose static lower bound is below 10 ms; from 10 ms,
    ceil(200 ms / lb) warm-ups, at least W and at most 6; off with long_warm_ms = 0."""
    sel = so.SelectorOracle(3, blocked=True)
    assert [sel.warm_count(x) for x in (0.0, 9.99e6, 10e6, 31.3e6, 62.5e6, 188e6, 250e6)] == [1, 1, 6, 6, 4, 2, 1]
    assert so.SelectorOracle(3, long_warm_ms=0).warm_count(50e6) == 1
    assert so.SelectorOracle(3, calib_warmup=3).warm_count(150e6) == 3      # never below W


def test_long_kernel_calibration_plan():
    """Blocked calibration of three long variants (lb 31 ms, 31 ms, 62.5 ms): 6 + 3, 6 + 3, then
    4 + 3 executions, warm-ups dropped, then model mode on the smallest timed mean."""
    sel = so.SelectorOracle(3, blocked=True, prune_pct=0)
    lb = [31e6, 31e6, 62.5e6]
    cost = [52_000_000, 50_000_000, 100_000_000]
    trace = []
    for _ in range(26):
        v, mode = sel.decide("k", [0, 1, 2], lb)
        warm = sel.commit(v, "k", mode, lb[v])
        sel.harvest(v, "k", mode, warm, cost[v])
        trace.append((v, mode))
    assert [v for v, _ in trace[:25]] == [0] * 9 + [1] * 9 + [2] * 7
    assert [m for _, m in trace[:9]] == [so.MODE_WARMUP] * 6 + [so.MODE_CALIB] * 3
    assert [m for _, m in trace[18:25]] == [so.MODE_WARMUP] * 4 + [so.MODE_CALIB] * 3
    assert trace[25] == (1, so.MODE_MODEL)
    assert sel.rec(0, "k").count == 3 and sel.rec(2, "k").count == 3
