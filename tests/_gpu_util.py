"""Shared helpers for the -m gpu tests: device-twin generator, tensor plumbing, sampled oracle."""
import ctypes
import os

import numpy as np

import gen

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
_gen_lib = None


def gen_lib():
    global _gen_lib
    if _gen_lib is None:
        lib = ctypes.CDLL(os.path.join(ROOT, "gen", "libcompar_gen.so"))
        lib.compar_gen_fill.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                        ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
        lib.compar_gen_fill.restype = ctypes.c_int
        _gen_lib = lib
    return _gen_lib


def device_matrix(tag, rows, cols, dist=gen.DIST_U, dtype="f32", seed=gen.SEED_DATA, transposed=False, ld=None):
    """Generate a logical rows x cols matrix on cuda:0 with the device twin.  Returns the
    storage tensor (cols x rows when transposed)."""
    import torch
    srows, scols = (cols, rows) if transposed else (rows, cols)
    ld = scols if ld is None else ld
    tdt = torch.float32 if dtype == "f32" else torch.bfloat16
    buf = torch.empty((srows, ld), dtype=tdt, device="cuda")
    rc = gen_lib().compar_gen_fill(buf.data_ptr(), 0 if dtype == "f32" else 1, rows, cols, ld, seed, tag, dist,
                                   1 if transposed else 0, torch.cuda.current_stream().cuda_stream)
    assert rc == 0, rc
    return buf[:, :scols] if ld != scols else buf


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
