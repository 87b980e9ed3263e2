"""Hypothesis-driven parity fuzzing on the GPU (-m gpu): random shapes (including non-multiples of
every tile size), leading-dimension padding, transB, alpha/beta (beta = 0 with NaN C_in), for every
eligible variant of a random precision class, checked against the FP64 oracle at the BASELINE
tolerances (1e-5 wherever no TF32 truncation applies) and element by element against the
FP32-accumulation bound.  Integer-valued inputs must be bitwise exact."""
import numpy as np
import pytest

import gen
from oracle import gemm as og

torch = pytest.importorskip("torch")
hyp = pytest.importorskip("hypothesis")
from hypothesis import HealthCheck, given, settings, strategies as st  # noqa: E402

pytestmark = pytest.mark.gpu

from tests._gpu_util import assert_parity, to_device, to_host_f64  # noqa: E402

cm = pytest.importorskip("paper_2311_03543_b200.compar")

# BF16: the oracle consumes the same BF16 values, only FP32 accumulation error remains;
# TF32 keeps 5e-3 only for its tensor-core variants (FFMA variants under COMPUTE_TF32 are exact FP32)
TOL = {cm.COMPUTE_F32_STRICT: 1e-5, cm.COMPUTE_TF32: 5e-3, cm.COMPUTE_BF16: 1e-5, cm.COMPUTE_F32_SPLIT: 1e-5}
_CTX = {}


def ctx():
    if "c" not in _CTX:
        _CTX["c"] = cm.Compar()
    return _CTX["c"]


@settings(max_examples=60, deadline=None, suppress_health_check=list(HealthCheck))
@given(m=st.integers(1, 700), n=st.integers(1, 700), k=st.integers(1, 900),
       compute=st.sampled_from([cm.COMPUTE_F32_STRICT, cm.COMPUTE_TF32, cm.COMPUTE_BF16, cm.COMPUTE_F32_SPLIT]),
       transB=st.integers(0, 1), pad=st.sampled_from([0, 8, 24]), beta=st.sampled_from([0.0, 0.5, -1.0]),
       integer=st.booleans(), seed=st.integers(0, 10 ** 6), pick=st.integers(0, 10))
def test_fuzz_parity(m, n, k, compute, transB, pad, beta, integer, seed, pick):
    _fuzz_case(m, n, k, compute, transB, pad, beta, integer, seed, pick)


@settings(max_examples=25, deadline=None, suppress_health_check=list(HealthCheck))
@given(m=st.integers(1, 300), n=st.integers(1, 300), k=st.integers(2000, 12000),
       compute=st.sampled_from([cm.COMPUTE_TF32, cm.COMPUTE_BF16, cm.COMPUTE_F32_SPLIT]),
       transB=st.integers(0, 1), pad=st.sampled_from([0, 8]), beta=st.sampled_from([0.0, 0.5]),
       integer=st.booleans(), seed=st.integers(0, 10 ** 6), pick=st.integers(0, 10))
def test_fuzz_parity_deep_k(m, n, k, compute, transB, pad, beta, integer, seed, pick):
    """Deep K (where the split-K variant becomes eligible), small M x N."""
    _fuzz_case(m, n, k, compute, transB, pad, beta, integer, seed, pick)


def _fuzz_case(m, n, k, compute, transB, pad, beta, integer, seed, pick):
    c = ctx()
    dtype_id = cm.BF16 if compute == cm.COMPUTE_BF16 else cm.F32
    dt = "bf16" if dtype_id == cm.BF16 else "f32"
    dist = gen.DIST_I if integer else gen.DIST_U
    A = gen.matrix(gen.TAG_A, m, k, dist, dt, seed=seed)
    B = gen.matrix(gen.TAG_B, k, n, dist, dt, seed=seed)
    C0 = gen.matrix(gen.TAG_C, m, n, dist, "f32", seed=seed)
    lda, ldb, ldc = k + pad, (k if transB else n) + pad, n + pad
    Ad = to_device(A, dt, lda)
    Bd = to_device(np.ascontiguousarray(B.T) if transB else B, dt, ldb)
    Cd = to_device(C0, "f32", ldc)
    if beta == 0.0:
        Cd.fill_(float("nan"))
    alpha = 2.0 if integer else 1.5
    d = cm.make_desc(m, n, k, A=Ad, B=Bd, C_in=Cd, C_out=Cd, lda=lda, ldb=ldb, ldc_in=ldc, ldc_out=ldc, alpha=alpha,
                     beta=beta, in_dtype=dtype_id, compute=compute, transB=transB)
    elig = []
    for v in range(len(c.variants())):
        d.variant_hint = v
        try:
            c.select(d)
            elig.append(v)
        except cm.ComparError:
            pass
    assert elig, "at least one variant must be eligible"
    d.variant_hint = elig[pick % len(elig)]
    r = c.run(d)
    assert r.status == 0
    got = to_host_f64(Cd[:, :n])
    ref = og.gemm(A, B, C0, alpha=alpha, beta=beta, dtype=dt)
    if integer:
        np.testing.assert_array_equal(got, ref)
    else:
        name = c.variants()[d.variant_hint][0]
        tf32 = name.startswith("tc_tf32")
        tol = TOL[compute] if tf32 or compute != cm.COMPUTE_TF32 else 1e-5
        # (tc_f32x3 claims FP32 accuracy: no tensor-core widening of the norm tolerance, R38)
        assert_parity(got, ref, A, B, C0, alpha, beta, dt, tf32, tol, (name, m, n, k),
                      tc=name.startswith("tc_") and name != "tc_f32x3")
