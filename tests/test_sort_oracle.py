"""Pins of the sort oracle (oracle/sort.py; NEXT-3, reading R24) — not against itself: IEEE
754 totalOrder worked example, a pairwise comparator written from the standard's prose with
brute force over all permutations, and reduction to numpy.sort where the orders coincide."""
import itertools

import numpy as np
import pytest

from oracle import sort as osort


def f32_bits(xs):
    return np.array(xs, dtype=np.float32).view(np.uint32)


def from_bits(bs):
    return np.array(bs, dtype=np.uint32).view(np.float32)


NEG_NAN = from_bits([0xFFC00000])[0]
POS_NAN = from_bits([0x7FC00000])[0]


def total_le(a, b):
    """IEEE 754-2008 §5.10 totalOrder(a, b) for binary32, from the prose: a negative sign orders
    before a positive one; among positives the larger magnitude (exponent, then significand —
    i.e. the larger 31-bit pattern) is larger; among negatives it is smaller."""
    ba, bb = int(f32_bits([a])[0]), int(f32_bits([b])[0])
    sa, sb = ba >> 31, bb >> 31
    if sa != sb:
        return sa == 1
    ma, mb = ba & 0x7FFFFFFF, bb & 0x7FFFFFFF
    return ma <= mb if sa == 0 else ma >= mb


def test_total_order_worked_example():
    keys = np.array([POS_NAN, -0.0, 1.0, -np.inf, 0.0, -1.0, np.inf, NEG_NAN, 1e-45, -1e-45], dtype=np.float32)
    want = [NEG_NAN, -np.inf, -1.0, -1e-45, -0.0, 0.0, 1e-45, 1.0, np.inf, POS_NAN]
    np.testing.assert_array_equal(f32_bits(osort.sort(keys)), f32_bits(want))


def test_brute_force_all_permutations():
    rng = np.random.default_rng(0)
    pool = np.array([0.0, -0.0, 1.5, -1.5, np.inf, -np.inf, POS_NAN, NEG_NAN, 2.0, 3e-40], dtype=np.float32)
    for _ in range(40):
        x = rng.choice(pool, size=rng.integers(1, 7))
        got = f32_bits(osort.sort(x))
        ok = [p for p in set(itertools.permutations(f32_bits(x).tolist()))
              if all(total_le(from_bits([p[i]])[0], from_bits([p[i + 1]])[0]) for i in range(len(p) - 1))]
        assert len(ok) == 1 and tuple(got.tolist()) == ok[0]


@pytest.mark.parametrize("kt", [osort.KEY_U32, osort.KEY_I32, osort.KEY_F32])
def test_reduces_to_numpy_sort(kt):
    rng = np.random.default_rng(kt)
    n = 100000
    if kt == osort.KEY_F32:     # no NaN and no -0: totalOrder == numeric order
        x = (rng.standard_normal(n) * 1e3).astype(np.float32)
        x[x == 0] = 1.0
    elif kt == osort.KEY_I32:
        x = rng.integers(-2 ** 31, 2 ** 31, n, dtype=np.int64).astype(np.int32)
    else:
        x = rng.integers(0, 2 ** 32, n, dtype=np.uint64).astype(np.uint32)
    np.testing.assert_array_equal(osort.sort(x, kt), np.sort(x))


def test_invariants():
    rng = np.random.default_rng(3)
    x = rng.standard_normal(5000).astype(np.float32)
    x[::7] = -0.0
    x[::11] = POS_NAN
    y = osort.sort(x)
    assert sorted(f32_bits(x).tolist()) == sorted(f32_bits(y).tolist())          # a permutation
    np.testing.assert_array_equal(f32_bits(osort.sort(y)), f32_bits(y))           # idempotent
    np.testing.assert_array_equal(f32_bits(osort.sort(x[::-1].copy())), f32_bits(y))
    assert osort.sort(np.zeros(0, np.float32)).size == 0
