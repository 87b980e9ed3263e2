"""ctypes front end of the device-twin generator (gen/gen.cu, include/compar_gen.h)."""
import ctypes
import os

from .inputs import DIST_U, SEED_DATA

_HERE = os.path.dirname(os.path.abspath(__file__))
_lib = None


def lib():
    global _lib
    if _lib is None:
        path = os.path.join(_HERE, "libcompar_gen.so")
        if not os.path.exists(path):
            raise ImportError(f"{path} not built (python -m paper_2311_03543_b200.build)")
        L = ctypes.CDLL(path)
        i64 = ctypes.c_int64
        L.compar_gen_fill.argtypes = [ctypes.c_void_p, ctypes.c_int, i64, i64, i64, i64, i64, ctypes.c_uint64,
                                      ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
        L.compar_gen_fill.restype = ctypes.c_int
        _lib = L
    return _lib


def fill(ptr, dtype, rows, cols, ld, tag, dist=DIST_U, seed=SEED_DATA, transposed=False, row0=0, col0=0,
         stream=None):
    """Asynchronously fill logical block [row0:row0+rows, col0:col0+cols] of matrix `tag` at `ptr`."""
    rc = lib().compar_gen_fill(ptr, 0 if dtype == "f32" else 1, rows, cols, ld, row0, col0, seed, tag, dist,
                               1 if transposed else 0, stream)
    if rc != 0:
        raise RuntimeError(f"compar_gen_fill failed ({rc})")


def device_matrix(tag, rows, cols, dist=DIST_U, dtype="f32", seed=SEED_DATA, transposed=False, ld=None, row0=0,
                  col0=0, device="cuda"):
    """torch tensor on `device` holding the logical block (stored transposed if asked)."""
    import torch
    srows, scols = (cols, rows) if transposed else (rows, cols)
    ld = scols if ld is None else ld
    buf = torch.empty((srows, ld), dtype=torch.float32 if dtype == "f32" else torch.bfloat16, device=device)
    fill(buf.data_ptr(), dtype, rows, cols, ld, tag, dist, seed, transposed, row0, col0,
         torch.cuda.current_stream().cuda_stream)
    return buf[:, :scols] if ld != scols else buf
