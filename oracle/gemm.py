"""ctypes front end of the FP64 oracle GEMM (oracle/gemm_oracle.c).

TEST INFRASTRUCTURE ONLY — see oracle/__init__.py.

`gemm(A, B, C_in, alpha, beta)` returns the FP64 result of
C_out = alpha * A @ B + beta * C_in.
Operands may be float32 arrays or uint16 BF16 bit patterns (dtype="bf16"); they
are widened EXACTLY to float64 here — the values the GPU consumes — and the
result stays FP64 (never rounded before comparison, reading R8).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gemm_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so (gcc -O2 -ffp-contract=off -fopenmp, no -march)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
                               "-fPIC", "-shared", "-o", _LIB + ".tmp", _SRC])
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB)
            d, lg, p = ctypes.c_double, ctypes.c_long, ctypes.c_void_p
            lib.compar_oracle_gemm.argtypes = [lg, lg, lg, d, p, lg, p, lg, d, p, lg, p, lg]
            lib.compar_oracle_gemm.restype = None
            lib.compar_oracle_threads.restype = ctypes.c_int
            lib.compar_oracle_set_threads.argtypes = [ctypes.c_int]
            lib.compar_oracle_set_threads.restype = None
            _lib = lib
    return _lib


def widen(x: np.ndarray, dtype: str = "f32") -> np.ndarray:
    """Exact widening of the consumed operand values to float64."""
    x = np.asarray(x)
    if dtype == "bf16" or x.dtype == np.uint16:
        x = (x.astype(np.uint32) << np.uint32(16)).view(np.float32)
    return np.ascontiguousarray(x, dtype=np.float64)


def gemm(A, B, C_in=None, alpha: float = 1.0, beta: float = 0.0, dtype: str = "f32") -> np.ndarray:
    """FP64 oracle: alpha * A @ B + beta * C_in with A (M x K), B (K x N), C_in (M x N)."""
    lib = _load()
    A64 = widen(A, dtype)
    B64 = widen(B, dtype)
    if A64.ndim != 2 or B64.ndim != 2 or A64.shape[1] != B64.shape[0]:
        raise ValueError(f"shape mismatch {A64.shape} x {B64.shape}")
    M, K = A64.shape
    N = B64.shape[1]
    out = np.empty((M, N), dtype=np.float64)
    if beta != 0.0:
        if C_in is None:
            raise ValueError("beta != 0 needs C_in")
        C64 = np.ascontiguousarray(np.asarray(C_in, dtype=np.float64))
        if C64.shape != (M, N):
            raise ValueError("C_in shape mismatch")
        cptr, ldc = C64.ctypes.data, N
    else:
        C64, cptr, ldc = None, None, max(N, 1)
    lib.compar_oracle_gemm(M, N, K, float(alpha),
                           A64.ctypes.data, max(K, 1), B64.ctypes.data, max(N, 1),
                           float(beta), cptr, ldc, out.ctypes.data, max(N, 1))
    return out


def threads() -> int:
    return int(_load().compar_oracle_threads())


def set_threads(n: int) -> None:
    """OpenMP threads for later oracle calls (timing only; results do not depend on it)."""
    _load().compar_oracle_set_threads(int(n))


U_F32 = 2.0 ** -24       # unit roundoff of FP32 round-to-nearest
DELTA_TF32 = 2.0 ** -10  # relative error of truncating an FP32 value to TF32 (10 explicit mantissa bits)


def elementwise_bound(A, B, C_in=None, alpha: float = 1.0, beta: float = 0.0, dtype: str = "f32",
                      tf32: bool = False, c: float = 2.0) -> np.ndarray:
    """Componentwise forward-error bound of C_out = alpha*A@B + beta*C_in computed with FP32
    accumulation in ANY summation order (the classical dot-product bound |fl(x.y) - x.y| <=
    gamma_K |x|.|y|, gamma_K ~ K*u; Higham, Accuracy and Stability of Numerical Algorithms §3.1):

        |C - C_exact| <= |alpha| * (e_op + c*K*u) * (1 + e_op + c*K*u) * (|A| @ |B|)
                         + 2u * (|alpha| * (1 + ...) * (|A| @ |B|) + |beta| * |C_in|)

    u = 2^-24.  Products of the consumed operands are exact in FP32 (FP32 x FP32 in an FMA, BF16 x
    BF16 and TF32 x TF32 fit 24 bits), so the operand term e_op is 0 except for TF32, whose
    hardware truncation of each operand (R6) perturbs every product by at most
    e_op = 2*2^-10 + 2^-20 relative.  c >= 1 widens K*u for accumulators that are not round-to-
    nearest (tensor-core block sums truncate after alignment); c = 2 by default.  The trailing 2u
    terms are the two roundings of the alpha/beta epilogue.  Returns the FP64 bound array.
    |A| @ |B| is this module's own FP64 GEMM of the absolute values."""
    A64, B64 = np.abs(widen(A, dtype)), np.abs(widen(B, dtype))
    K = A64.shape[1]
    e_op = (2.0 * DELTA_TF32 + DELTA_TF32 ** 2) if tf32 else 0.0
    acc = e_op + c * K * U_F32
    absab = gemm(A64.astype(np.float64), B64.astype(np.float64)) if K > 0 else np.zeros((A64.shape[0], B64.shape[1]))
    grow = abs(alpha) * (1.0 + acc) * absab
    bound = abs(alpha) * acc * (1.0 + acc) * absab + 2.0 * U_F32 * grow
    if beta != 0.0:
        bound = bound + 2.0 * U_F32 * abs(beta) * np.abs(np.asarray(C_in, dtype=np.float64))
    return bound


def elementwise_violation(c_test, c_ref, bound) -> float:
    """max_ij |C - C_ref| / bound_ij (<= 1 means every element is inside its bound; a zero bound
    requires an exact match)."""
    diff = np.abs(np.asarray(c_test, dtype=np.float64) - np.asarray(c_ref, dtype=np.float64))
    bound = np.asarray(bound, dtype=np.float64)
    if diff.size == 0:
        return 0.0
    exact = bound == 0.0
    if np.any(diff[exact] != 0.0) or not np.all(np.isfinite(diff)):
        return float("inf")
    return float(np.max(np.where(exact, 0.0, diff / np.where(exact, 1.0, bound))))


def rel_fro(c_test, c_ref) -> float:
    """max-relative-Frobenius metric of BASELINE.json: ||C - C_ref||_F / ||C_ref||_F (FP64).

    If ||C_ref||_F == 0 the result is 0.0 only when C is exactly zero, else inf
    (reading R8)."""
    c_test = np.asarray(c_test, dtype=np.float64)
    c_ref = np.asarray(c_ref, dtype=np.float64)
    den = np.linalg.norm(c_ref)
    num = np.linalg.norm(c_test - c_ref)
    if den == 0.0:
        return 0.0 if num == 0.0 else float("inf")
    return float(num / den)
