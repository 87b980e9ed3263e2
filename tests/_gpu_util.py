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


def assert_parity(got, ref, A, B, C0, alpha, beta, dtype, tf32, tol, what=""):
    """The two parity checks against the FP64 oracle: the BASELINE max relative Frobenius error
    (<= tol) AND the componentwise FP32-accumulation bound of oracle.gemm.elementwise_bound on
    every element (so a handful of wrong elements cannot hide inside a small norm ratio)."""
    from oracle import gemm as og
    err = og.rel_fro(got, ref)
    assert err <= tol, (what, "rel_fro", err, tol)
    bound = og.elementwise_bound(A, B, C0, alpha, beta, dtype=dtype, tf32=tf32)
    v = og.elementwise_violation(got, ref, bound)
    assert v <= 1.0, (what, "elementwise bound exceeded by", v)
    return err
