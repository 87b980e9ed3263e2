"""Pins of the shared input generator (gen/) — SURVEY.md §8(d) recipe."""
import numpy as np

import gen


def test_splitmix64_published_vector(golden):
    g = golden("splitmix64.txt")
    seed = int(g["seed"])
    expected = [int(k) for k in g if k not in ("seed",)]
    gamma = 0x9E3779B97F4A7C15
    states = np.array([(seed + n * gamma) & (2 ** 64 - 1) for n in range(5)], dtype=np.uint64)
    assert [int(x) for x in gen.splitmix64(states)] == expected


def test_distributions_exact_and_in_range():
    h = gen.splitmix64(np.arange(100000, dtype=np.uint64))
    u = gen.values_f32(h, gen.DIST_U)
    assert u.min() >= -1.0 and u.max() < 1.0
    # exact in FP32: value * 2^23 is an integer
    assert np.all(np.floor(u.astype(np.float64) * 2 ** 23) == u.astype(np.float64) * 2 ** 23)
    p = gen.values_f32(h, gen.DIST_P)
    assert p.min() >= 0.0 and p.max() < 1.0
    i = gen.values_f32(h, gen.DIST_I)
    assert set(np.unique(i).tolist()) == {-2.0, -1.0, 0.0, 1.0, 2.0}
    assert abs(u.mean()) < 0.01 and abs(p.mean() - 0.5) < 0.01


def test_bf16_rne_ties_and_exact_values():
    x = np.array([1.0, 1.00390625, 1.01171875, -2.5, 3.0e-3], dtype=np.float32)
    # 1 + 2^-8 is a tie between 1.0 and 1 + 2^-7 -> even (1.0); 1 + 3*2^-8 ties -> 1 + 2^-6 (even)
    b = gen.f32_to_bf16_bits_rne(x)
    assert b[0] == 0x3F80 and b[1] == 0x3F80 and b[2] == 0x3F82
    assert gen.bf16_bits_to_f32(b[3:4])[0] == -2.5
    # round-trip of representable values is the identity
    vals = gen.bf16_bits_to_f32(np.arange(0x3F00, 0x4100, dtype=np.uint16))
    assert np.array_equal(gen.f32_to_bf16_bits_rne(vals), np.arange(0x3F00, 0x4100, dtype=np.uint16))


def test_logical_indexing_consistent():
    """rows/cols/entries are views of the same logical matrix (used by sampled parity)."""
    full = gen.matrix(gen.TAG_B, 40, 50, gen.DIST_U, "bf16")
    rows = [0, 7, 39]
    cols = [1, 2, 49]
    assert np.array_equal(gen.matrix_rows(gen.TAG_B, rows, 50, dtype="bf16"), full[rows])
    assert np.array_equal(gen.matrix_cols(gen.TAG_B, 40, cols, dtype="bf16"), full[:, cols])
    assert np.array_equal(gen.matrix_entries(gen.TAG_B, rows, cols, dtype="bf16"), full[np.ix_(rows, cols)])


def test_tags_and_seeds_differ():
    a = gen.matrix(gen.TAG_A, 8, 8)
    b = gen.matrix(gen.TAG_B, 8, 8)
    a2 = gen.matrix(gen.TAG_A, 8, 8, seed=gen.SEED_DATA + 1)
    assert not np.array_equal(a, b) and not np.array_equal(a, a2)
