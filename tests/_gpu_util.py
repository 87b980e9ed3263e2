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
