"""Shared helpers for the -m gpu tests: device-twin generator, tensor plumbing."""
import numpy as np

from gen.device import device_matrix  # noqa: F401


def to_device(arr, dtype="f32", ld=None):
    """Host numpy (float32 or uint16 bf16 bits) -> cuda tensor with optional padded leading dim."""
    import torch
    rows, cols = arr.shape
    ld = cols if ld is None else ld
    if dtype == "bf16":
        t = torch.from_numpy(np.ascontiguousarray(arr).view(np.int16)).view(torch.bfloat16)
        buf = torch.zeros((rows, ld), dtype=torch.bfloat16, device="cuda")
    else:
        t = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float32))
        buf = torch.zeros((rows, ld), dtype=torch.float32, device="cuda")
    buf[:, :cols].copy_(t.cuda())
    return buf


def to_host_f64(t):
    return t.float().cpu().numpy().astype(np.float64)


def tc_accum_tol(k):
    """rel-Fro tolerance of a tensor-core variant whose operands the oracle consumes exactly (BF16):
    the tcgen05 FP32 accumulator is not round-to-nearest — measured 3.7e-5 at K = 32768 on
    U(-1,1) against 3.2e-6 for a simulated round-to-nearest FP32 sum (R33) — so the
    bound grows like one truncation of 2^-23 per K = 16 MMA step: K/16 * 2^-23 = K * 2^-27, and
    never below the strict-FP32 1e-5."""
    return max(1e-5, k * 2.0 ** -27)


def assert_parity(got, ref, A, B, C0, alpha, beta, dtype, tf32, tol, what="", tc=False):
    """The two parity checks against the FP64 oracle: the BASELINE max relative Frobenius error
    (<= tol; for tensor-core variants without TF32 truncation at least tc_accum_tol(K)) AND the
    componentwise FP32-accumulation bound of oracle.gemm.elementwise_bound on every element (so a
    handful of wrong elements cannot hide inside a small norm ratio)."""
    from oracle import gemm as og
    if tc and not tf32:
        tol = max(tol, tc_accum_tol(np.asarray(A).shape[1]))
    err = og.rel_fro(got, ref)
    bound = og.elementwise_bound(A, B, C0, alpha, beta, dtype=dtype, tf32=tf32)
    v = og.elementwise_violation(got, ref, bound)
    # (R8: below 64 output elements the norm ratio degenerates into a few elements' relative errors,
    # which cancellation in a dot product can make arbitrarily large — there the componentwise bound
    # alone is the criterion; found by the fuzz test at m = n = 1, K = 2000: 4.7e-5, bound met)
    norm_ok = err <= tol or np.size(got) < 64
    assert norm_ok and v <= 1.0, (what, "rel_fro", err, "tol", tol, "elementwise violation", v)
    return err
