"""Canonical host-side counter-based input generator (numpy).

Recipe (SURVEY.md §8(d) "Inputs"):

    h = splitmix64(seed ^ (tag << 56) ^ (i << 28) ^ j)        i = row, j = column
    U = ((h >> 40) - 2**23) * 2**-23     in [-1, 1), exact in FP32     (primary)
    P =  (h >> 40)          * 2**-24     in [ 0, 1), exact in FP32     (Rodinia-like)
    I =   h mod 5 - 2                    in {-2..2}, exact everywhere  (exactness runs)

BF16 inputs are the round-to-nearest-even quantisation of the FP32 value; the
quantised bits are what both sides consume.

Indices are LOGICAL: B[k][n] has the same value whether B is stored K x N or
transposed (N x K), so the transB path is fed the same matrix.

`splitmix64` is Steele/Lea/Flood's finaliser as published by Vigna
(x += 0x9E3779B97F4A7C15; two xor-shift-multiply rounds; final xor-shift);
tests/golden/splitmix64.txt pins it to the published test vector.
This module contains no GEMM arithmetic (task rule: generator is shared, the
method is not).
"""
from __future__ import annotations

import numpy as np

DIST_U, DIST_P, DIST_I = 0, 1, 2
TAG_A, TAG_B, TAG_C = 1, 2, 3
SEED_DATA = 20231106
SEED_STREAM = 7

_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """splitmix64 output for state x (the value returned by next() after x += gamma)."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + _GAMMA
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def counters(seed: int, tag: int, i: np.ndarray, j: np.ndarray) -> np.ndarray:
    """Counter word for element (i, j) of matrix `tag`; broadcasts i against j."""
    i = np.asarray(i, dtype=np.uint64)
    j = np.asarray(j, dtype=np.uint64)
    base = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) ^ (np.uint64(tag) << np.uint64(56))
    return base ^ (i << np.uint64(28)) ^ j


def values_f32(h: np.ndarray, dist: int) -> np.ndarray:
    """Map hash words to FP32 values of distribution `dist` (all exact in FP32)."""
    if dist == DIST_U:
        r = (h >> np.uint64(40)).astype(np.int64) - (1 << 23)
        return (r.astype(np.float64) * 2.0 ** -23).astype(np.float32)
    if dist == DIST_P:
        r = (h >> np.uint64(40)).astype(np.int64)
        return (r.astype(np.float64) * 2.0 ** -24).astype(np.float32)
    if dist == DIST_I:
        return ((h % np.uint64(5)).astype(np.int64) - 2).astype(np.float32)
    raise ValueError(f"unknown distribution {dist}")


def f32_to_bf16_bits_rne(x: np.ndarray) -> np.ndarray:
    """Round FP32 to BF16 (nearest, ties to even); returns the 16-bit patterns.

    Inputs here are finite (the generator never produces NaN/Inf)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    lsb = (u >> np.uint32(16)) & np.uint32(1)
    with np.errstate(over="ignore"):
        r = u + np.uint32(0x7FFF) + lsb
    return (r >> np.uint32(16)).astype(np.uint16)


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    """Exact widening of BF16 bit patterns to FP32."""
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def values_bf16_bits(h: np.ndarray, dist: int) -> np.ndarray:
    return f32_to_bf16_bits_rne(values_f32(h, dist))


def _convert(h: np.ndarray, dist: int, dtype: str) -> np.ndarray:
    if dtype == "f32":
        return values_f32(h, dist)
    if dtype == "bf16":
        return values_bf16_bits(h, dist)
    raise ValueError(f"unknown dtype {dtype}")


def matrix(tag: int, rows: int, cols: int, dist: int = DIST_U, dtype: str = "f32",
           seed: int = SEED_DATA) -> np.ndarray:
    """Logical rows x cols matrix: float32 values ("f32") or uint16 BF16 bits ("bf16")."""
    i = np.arange(rows, dtype=np.uint64)[:, None]
    j = np.arange(cols, dtype=np.uint64)[None, :]
    return _convert(splitmix64(counters(seed, tag, i, j)), dist, dtype)


def matrix_rows(tag: int, row_idx, cols: int, dist: int = DIST_U, dtype: str = "f32",
                seed: int = SEED_DATA) -> np.ndarray:
    """Selected logical rows (len(row_idx) x cols) of matrix `tag`."""
    i = np.asarray(row_idx, dtype=np.uint64)[:, None]
    j = np.arange(cols, dtype=np.uint64)[None, :]
    return _convert(splitmix64(counters(seed, tag, i, j)), dist, dtype)


def matrix_cols(tag: int, rows: int, col_idx, dist: int = DIST_U, dtype: str = "f32",
                seed: int = SEED_DATA) -> np.ndarray:
    """Selected logical columns (rows x len(col_idx)) of matrix `tag`."""
    i = np.arange(rows, dtype=np.uint64)[:, None]
    j = np.asarray(col_idx, dtype=np.uint64)[None, :]
    return _convert(splitmix64(counters(seed, tag, i, j)), dist, dtype)


def matrix_entries(tag: int, row_idx, col_idx, dist: int = DIST_U, dtype: str = "f32",
                   seed: int = SEED_DATA) -> np.ndarray:
    """Sub-matrix at the cross product row_idx x col_idx."""
    i = np.asarray(row_idx, dtype=np.uint64)[:, None]
    j = np.asarray(col_idx, dtype=np.uint64)[None, :]
    return _convert(splitmix64(counters(seed, tag, i, j)), dist, dtype)
