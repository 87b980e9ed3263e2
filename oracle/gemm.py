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
