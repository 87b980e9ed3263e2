"""The arithmetic claim behind the F32_SPLIT class (R38), checked on the CPU from its
definition (not from the GPU code): with hi = RN_tf32(x) and lo = RN_tf32(x - hi) (TF32 = FP32
with the low 13 mantissa bits zero, round to nearest even), every FP32 product satisfies

    |a*b - (hi_a*hi_b + hi_a*lo_b + lo_a*hi_b)| <= 3 * 2^-22 * |a*b|

and hi, lo are exact TF32 values (so a tensor core reading them as TF32 loses nothing).  That
per-product bound is what places the variant inside the FP32 dot-product bound from K >= 64.
"""
import numpy as np


def tf32_rn(x):
    """Round-to-nearest-even onto the TF32 grid, written from the format's definition: clear the low
    13 of FP32's 23 mantissa bits, rounding the dropped part to nearest with ties to even."""
    u = np.asarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    lsb = (u >> 13) & 1
    r = (u + 0x0FFF + lsb) & 0xFFFFE000
    return r.astype(np.uint32).view(np.float32)


def split(x):
    hi = tf32_rn(x)
    lo = tf32_rn((x.astype(np.float32) - hi).astype(np.float32))   # x - hi is exact in FP32
    return hi, lo


def rand_floats(rng, n, emin=-60, emax=60):
    m = rng.uniform(1.0, 2.0, n)
    e = rng.integers(emin, emax, n)
    s = rng.choice([-1.0, 1.0], n)
    return (s * m * np.exp2(e)).astype(np.float32)


def test_split_parts_are_tf32_and_exact_subtraction():
    rng = np.random.default_rng(0)
    x = rand_floats(rng, 200_000)
    hi, lo = split(x)
    assert not np.any(hi.view(np.uint32) & 0x1FFF)
    assert not np.any(lo.view(np.uint32) & 0x1FFF)
    # x - hi is representable: recomputing it in FP64 gives the same FP32 value
    d32 = (x - hi).astype(np.float32)
    np.testing.assert_array_equal(d32.astype(np.float64), x.astype(np.float64) - hi.astype(np.float64))
    # hi carries x to 2^-11 relative, hi + lo to 2^-22
    rel = np.abs(x.astype(np.float64) - hi - lo) / np.abs(x.astype(np.float64))
    assert rel.max() <= 2.0 ** -22


def test_three_product_error_bound():
    rng = np.random.default_rng(1)
    a = rand_floats(rng, 500_000)
    b = rand_floats(rng, 500_000)
    ha, la = split(a)
    hb, lb = split(b)
    f = lambda v: v.astype(np.float64)  # noqa: E731
    approx = f(ha) * f(hb) + f(ha) * f(lb) + f(la) * f(hb)        # the three TF32 products, exactly
    exact = f(a) * f(b)
    rel = np.abs(approx - exact) / np.abs(exact)
    assert rel.max() <= 3 * 2.0 ** -22, rel.max()
    # and the dropped term is the dominant one: without hi*lo + lo*hi the error is ~2^-11
    rel1 = np.abs(f(ha) * f(hb) - exact) / np.abs(exact)
    assert rel1.max() > 2.0 ** -13


def test_tf32_rounding_worked_examples():
    """Ties to even and carries, from the bit patterns: 1 + 2^-11 is a tie between 1 and 1 + 2^-10
    (even mantissa -> 1); 1 + 3*2^-11 is a tie between 1 + 2^-10 and 1 + 2^-9 (-> 1 + 2^-9);
    2 - 2^-23 rounds up across the exponent to 2."""
    ex = np.array([1 + 2.0 ** -11, 1 + 3 * 2.0 ** -11, 2 - 2.0 ** -23, 1 + 2.0 ** -10 + 2.0 ** -12], dtype=np.float32)
    want = np.array([1.0, 1 + 2.0 ** -9, 2.0, 1 + 2.0 ** -10], dtype=np.float32)
    np.testing.assert_array_equal(tf32_rn(ex), want)
