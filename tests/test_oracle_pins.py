"""Pins of the FP64 oracle GEMM against things other than itself (-m "not gpu").

Each test names the kind of pin (worked example / closed form / brute force /
library special case / invariant) and what plausible oracle bug it catches.
The oracle follows PAPER.md P:76-80, P:201-205 read as xGEMM (R1, R3).
"""
from fractions import Fraction

import numpy as np
import pytest

import gen
from oracle import gemm as og


@pytest.mark.parametrize("name", ["gemm_2x2.txt", "gemm_3x3_alpha_beta.txt", "gemm_rect_2x3x4.txt"])
def test_worked_examples(golden, name):
    """Worked examples (tests/golden): exact. Catches transposed operand, dropped alpha/beta."""
    g = golden(name)
    alpha, beta = float(g["alpha"]), float(g["beta"])
    out = og.gemm(g["A"].astype(np.float32), g["B"].astype(np.float32),
                  g.get("C_in"), alpha=alpha, beta=beta)
    np.testing.assert_array_equal(out, g["C_out"])


def _u(tag, r, c, seed=11):
    return gen.matrix(tag, r, c, gen.DIST_U, "f32", seed=seed)


def test_identity_closed_form():
    """A = I  =>  C = alpha*B + beta*C_in exactly (one nonzero product per element)."""
    M = 37
    B, C0 = _u(2, M, 53), _u(3, M, 53)
    A = np.eye(M, dtype=np.float32)
    out = og.gemm(A, B, C0, alpha=1.5, beta=0.5)
    ref = 1.5 * B.astype(np.float64) + 0.5 * C0.astype(np.float64)
    np.testing.assert_array_equal(out, ref)


def test_diagonal_closed_form():
    """A = diag(d)  =>  C[i][j] = alpha*d_i*B[i][j] + beta*C_in[i][j]. Catches row/col index swaps."""
    M, N = 29, 41
    d = _u(1, 1, M)[0]
    B, C0 = _u(2, M, N), _u(3, M, N)
    out = og.gemm(np.diag(d), B, C0, alpha=-2.0, beta=0.25)
    ref = -2.0 * (d.astype(np.float64)[:, None] * B.astype(np.float64)) + 0.25 * C0.astype(np.float64)
    np.testing.assert_array_equal(out, ref)


def test_rank1_and_ones_closed_form():
    """A = u 1^T, B = 1 v^T  =>  AB = K u_i v_j; all-ones => alpha*K + beta*C_in. Catches a dropped k term."""
    M, N, K = 9, 14, 33
    u = gen.matrix(1, M, 1, gen.DIST_I, "f32", seed=3)[:, 0]
    v = gen.matrix(2, 1, N, gen.DIST_I, "f32", seed=3)[0]
    A = np.repeat(u[:, None], K, axis=1)
    B = np.repeat(v[None, :], K, axis=0)
    out = og.gemm(A, B, alpha=1.0, beta=0.0)
    np.testing.assert_array_equal(out, K * np.outer(u, v).astype(np.float64))
    C0 = gen.matrix(3, M, N, gen.DIST_I, "f32", seed=3)
    out1 = og.gemm(np.ones((M, K), np.float32), np.ones((K, N), np.float32), C0, alpha=2.0, beta=-1.0)
    np.testing.assert_array_equal(out1, 2.0 * K - C0.astype(np.float64))


def test_exact_rational_brute_force():
    """Brute force with fractions.Fraction on random FP32 inputs, M,N,K <= 7:
    the FP64 oracle is within K * 2^-52 * sum|terms| of the exact value."""
    rng = np.random.default_rng(5)
    for trial in range(12):
        M, N, K = rng.integers(1, 8, size=3)
        A = _u(1, M, K, seed=100 + trial)
        B = _u(2, K, N, seed=100 + trial)
        C0 = _u(3, M, N, seed=100 + trial)
        alpha, beta = 1.5, -0.75
        out = og.gemm(A, B, C0, alpha=alpha, beta=beta)
        for i in range(M):
            for j in range(N):
                exact = Fraction(alpha) * sum(Fraction(float(A[i, k])) * Fraction(float(B[k, j]))
                                              for k in range(K)) + Fraction(beta) * Fraction(float(C0[i, j]))
                mag = abs(alpha) * sum(abs(float(A[i, k]) * float(B[k, j])) for k in range(K)) \
                    + abs(beta * float(C0[i, j]))
                assert abs(Fraction(out[i, j]) - exact) <= Fraction((K + 2) * 2.0 ** -52 * mag + 1e-300)


def test_integer_inputs_exact():
    """I-distribution inputs: every partial sum is an integer < 2^53, so the oracle is exact;
    compared with Python integer arithmetic."""
    M, N, K = 13, 17, 300
    A = gen.matrix(1, M, K, gen.DIST_I, "f32")
    B = gen.matrix(2, K, N, gen.DIST_I, "f32")
    C0 = gen.matrix(3, M, N, gen.DIST_I, "f32")
    out = og.gemm(A, B, C0, alpha=2.0, beta=-1.0)
    Ai, Bi, Ci = A.astype(np.int64), B.astype(np.int64), C0.astype(np.int64)
    ref = 2 * (Ai @ Bi) - Ci
    np.testing.assert_array_equal(out, ref.astype(np.float64))


def test_numpy_float64_crosscheck():
    """Library special case: numpy float64 matmul on the widened inputs (rel <= 1e-13)."""
    M, N, K = 67, 45, 129
    A, B, C0 = _u(1, M, K), _u(2, K, N), _u(3, M, N)
    out = og.gemm(A, B, C0, alpha=1.5, beta=0.5)
    ref = 1.5 * (A.astype(np.float64) @ B.astype(np.float64)) + 0.5 * C0.astype(np.float64)
    assert og.rel_fro(out, ref) <= 1e-13


def test_bf16_widening_is_exact():
    """BF16 operands are widened exactly (bits << 16): same result as feeding the FP32 values."""
    M, N, K = 8, 9, 40
    Ab = gen.matrix(1, M, K, dtype="bf16")
    Bb = gen.matrix(2, K, N, dtype="bf16")
    out_b = og.gemm(Ab, Bb, dtype="bf16")
    out_f = og.gemm(gen.bf16_bits_to_f32(Ab), gen.bf16_bits_to_f32(Bb))
    np.testing.assert_array_equal(out_b, out_f)


def test_beta_zero_does_not_read_c():
    """BLAS rule (R3): beta == 0 => C_in is not read; NaN in C_in must not propagate."""
    A, B = _u(1, 6, 7), _u(2, 7, 5)
    C0 = np.full((6, 5), np.nan, dtype=np.float32)
    out = og.gemm(A, B, C0, alpha=1.5, beta=0.0)
    assert np.isfinite(out).all()
    np.testing.assert_array_equal(out, og.gemm(A, B, alpha=1.5, beta=0.0))


def test_alpha_zero_and_k_zero():
    """BLAS rule (R3): alpha == 0 => A, B unread, C = beta*C_in; K == 0 => C = beta*C_in."""
    A = np.full((4, 3), np.nan, dtype=np.float32)
    B = np.full((3, 5), np.inf, dtype=np.float32)
    C0 = _u(3, 4, 5)
    out = og.gemm(A, B, C0, alpha=0.0, beta=0.5)
    np.testing.assert_array_equal(out, 0.5 * C0.astype(np.float64))
    out_k0 = og.gemm(np.zeros((4, 0), np.float32), np.zeros((0, 5), np.float32), C0, alpha=1.5, beta=-2.0)
    np.testing.assert_array_equal(out_k0, -2.0 * C0.astype(np.float64))


def test_empty_m_n():
    assert og.gemm(np.zeros((0, 3), np.float32), _u(2, 3, 4)).shape == (0, 4)
    assert og.gemm(_u(1, 4, 3), np.zeros((3, 0), np.float32)).shape == (4, 0)


def test_transpose_identity():
    """Invariant: (alpha A B + beta C)^T = alpha B^T A^T + beta C^T, bit-exact (same k order,
    commutative products). Catches a transposed operand or an ld/stride mix-up."""
    M, N, K = 23, 31, 47
    A, B, C0 = _u(1, M, K), _u(2, K, N), _u(3, M, N)
    out = og.gemm(A, B, C0, alpha=1.5, beta=0.5)
    out_t = og.gemm(np.ascontiguousarray(B.T), np.ascontiguousarray(A.T), np.ascontiguousarray(C0.T),
                    alpha=1.5, beta=0.5)
    np.testing.assert_array_equal(out, out_t.T)


def test_rel_fro_metric():
    """The tolerance metric (R8): exact zero reference requires exact zero output."""
    assert og.rel_fro(np.zeros(3), np.zeros(3)) == 0.0
    assert og.rel_fro(np.ones(3), np.zeros(3)) == float("inf")
    assert og.rel_fro([3.0, 4.0], [0.0, 5.0]) == pytest.approx(np.sqrt(10.0) / 5.0)


def _fp32_sequential(A, B, C0, alpha, beta, tf32=False):
    """Independent simulation of an FP32 kernel: operands optionally truncated to TF32 (low 13
    mantissa bits cleared), every k-step one FMA acc = fl32(acc + a*b) (the product of two FP32
    values is exact in FP64), epilogue fl32(fl32(alpha*acc) + fl32(beta*c))."""
    def trunc(x):
        x = np.ascontiguousarray(x, dtype=np.float32)
        return (x.view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32) if tf32 else x
    a, b = trunc(A).astype(np.float64), trunc(B).astype(np.float64)
    acc = np.zeros((a.shape[0], b.shape[1]), dtype=np.float32)
    for k in range(a.shape[1]):
        acc = (acc.astype(np.float64) + np.outer(a[:, k], b[k, :])).astype(np.float32)
    out = (np.float32(alpha) * acc).astype(np.float32)
    if beta != 0.0:
        out = (out.astype(np.float64) + (np.float32(beta) * C0.astype(np.float32)).astype(np.float64)).astype(np.float32)
    return out.astype(np.float64)


@pytest.mark.parametrize("dist", [gen.DIST_U, gen.DIST_P])
def test_elementwise_bound_holds_for_fp32_accumulation(dist):
    """Error bound (Higham §3.1 dot-product bound, oracle/gemm.elementwise_bound): a simulated FP32
    sequential-FMA GEMM stays inside the componentwise bound at c = 1 (round-to-nearest), with the
    P distribution (all terms positive: the bound's worst case for bias)."""
    M, N, K = 12, 10, 2048
    A = gen.matrix(1, M, K, dist, "f32", seed=21)
    B = gen.matrix(2, K, N, dist, "f32", seed=21)
    C0 = gen.matrix(3, M, N, dist, "f32", seed=21)
    sim = _fp32_sequential(A, B, C0, 1.5, 0.5)
    ref = og.gemm(A, B, C0, alpha=1.5, beta=0.5)
    v = og.elementwise_violation(sim, ref, og.elementwise_bound(A, B, C0, 1.5, 0.5, c=1.0))
    assert 0.0 < v <= 1.0


def test_elementwise_bound_tf32_operand_term():
    """TF32 truncation (R6): the simulated TF32 GEMM is inside the bound only WITH the operand term
    e_op = 2*2^-10 + 2^-20 (catches a dropped e_op)."""
    M, N, K = 8, 9, 256
    A = gen.matrix(1, M, K, gen.DIST_P, "f32", seed=4)
    B = gen.matrix(2, K, N, gen.DIST_P, "f32", seed=4)
    sim = _fp32_sequential(A, B, None, 1.0, 0.0, tf32=True)
    ref = og.gemm(A, B)
    assert og.elementwise_violation(sim, ref, og.elementwise_bound(A, B, tf32=True, c=1.0)) <= 1.0
    assert og.elementwise_violation(sim, ref, og.elementwise_bound(A, B, tf32=False, c=1.0)) > 1.0


def test_elementwise_bound_catches_dropped_term_and_wrong_element():
    """A plausible kernel bug — one k-term dropped from one element, or one garbage element —
    fails the componentwise check although the Frobenius ratio of the whole matrix stays small."""
    M, N, K = 64, 64, 512
    A = gen.matrix(1, M, K, gen.DIST_U, "f32", seed=8)
    B = gen.matrix(2, K, N, gen.DIST_U, "f32", seed=8)
    ref = og.gemm(A, B)
    bound = og.elementwise_bound(A, B)
    bad = ref.copy()
    big = int(np.argmax(np.abs(A[5].astype(np.float64) * B[:, 7].astype(np.float64))))
    bad[5, 7] -= float(A[5, big]) * float(B[big, 7])       # dropped k-term
    assert og.elementwise_violation(bad, ref, bound) > 1.0
    bad2 = ref.copy()
    bad2[10, 3] = 0.0                                         # one unwritten element
    assert og.elementwise_violation(bad2, ref, bound) > 1.0
    assert og.rel_fro(bad2, ref) < 0.05
    assert og.elementwise_violation(ref, ref, bound) == 0.0


def test_elementwise_bound_k_zero_and_exact_zero():
    """K = 0: C = beta*C_in, the bound is the epilogue rounding only; a zero bound demands exactness."""
    C0 = _u(3, 4, 5)
    b = og.elementwise_bound(np.zeros((4, 0), np.float32), np.zeros((0, 5), np.float32), C0, 1.5, -2.0)
    np.testing.assert_allclose(b, 2.0 ** -23 * 2.0 * np.abs(C0.astype(np.float64)))
    z = np.zeros((2, 2))
    assert og.elementwise_violation(z, z, z) == 0.0
    assert og.elementwise_violation(z + 1e-30, z, z) == float("inf")
