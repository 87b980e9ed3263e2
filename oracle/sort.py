"""Sort oracle (a second interface through the same registry) — TEST
INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md P:76-78: "the sort function, two parameters are utilized: an array of floats and a scalar
integer" (Listing 1 is lost); P:60 names variants such as "bubble_sort", "merge_sort".  Reading
R24: sort(arr, n) rearranges arr[0..n) IN PLACE into ascending order.  Keys are FP32
(the paper's interface) or, for generality, uint32 / int32.  For FP32 the order is IEEE 754-2008
totalOrder (§5.10): -NaN < -Inf < ... < -0 < +0 < ... < +Inf < +NaN, NaNs ordered by payload, so
every input has exactly one sorted output (bit patterns compared, not just values).

The oracle is the definition: a stable sort by a comparison key that spells totalOrder out as
(sign, magnitude) — negative keys map to -1 - magnitude, positive ones to +magnitude — using the
library primitive numpy.argsort(kind="stable").  Independent of the CUDA radix transform.
"""
import numpy as np

KEY_U32, KEY_I32, KEY_F32 = 0, 1, 2
DTYPES = {KEY_U32: np.uint32, KEY_I32: np.int32, KEY_F32: np.float32}


def order_key(keys: np.ndarray, key_type: int) -> np.ndarray:
    """int64 array whose natural order is the key order of `key_type`."""
    if key_type == KEY_U32:
        return keys.astype(np.uint32).astype(np.int64)
    if key_type == KEY_I32:
        return keys.astype(np.int32).astype(np.int64)
    bits = np.ascontiguousarray(keys, dtype=np.float32).view(np.uint32).astype(np.int64)
    neg = (bits >> 31) == 1
    mag = bits & 0x7FFFFFFF
    return np.where(neg, -1 - mag, mag)


def sort(keys: np.ndarray, key_type: int = KEY_F32) -> np.ndarray:
    """Ascending (totalOrder for FP32) copy of `keys`, bit patterns preserved."""
    keys = np.ascontiguousarray(keys, dtype=DTYPES[key_type])
    return keys[np.argsort(order_key(keys, key_type), kind="stable")]
