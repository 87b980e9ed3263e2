"""Quick per-variant timing probe (development aid; bench.py is the measured contract)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import gen  # noqa: E402
from paper_2311_03543_b200 import compar as cm  # noqa: E402
from gen.device import device_matrix  # noqa: E402


def time_variant(ctx, name, m, n, k, reps=10, transB=0):
    names = [v for v, _ in ctx.variants()]
    vid = names.index(name)
    bf = "bf16" in name
    dt = "bf16" if bf else "f32"
    A = device_matrix(gen.TAG_A, m, k, dtype=dt)
    B = device_matrix(gen.TAG_B, k, n, dtype=dt, transposed=bool(transB))
    Cd = device_matrix(gen.TAG_C, m, n)
    d = cm.make_desc(m, n, k, A=A, B=B, C_in=Cd, C_out=Cd, alpha=1.5, beta=0.5,
                     in_dtype=cm.BF16 if bf else cm.F32,
                     compute=cm.COMPUTE_BF16 if bf else (cm.COMPUTE_TF32 if "tf32" in name else cm.COMPUTE_F32_STRICT),
                     transB=transB, variant_hint=vid, ldb=(k if transB else n))
    for _ in range(3):
        ctx.run(d)
    ns = sorted(ctx.run(d).ns for _ in range(reps))
    med = ns[len(ns) // 2]
    return med, 2.0 * m * n * k / med / 1e3


if __name__ == "__main__":
    ctx = cm.Compar()
    cases = [("tc_bf16_2sm_w", 8192, 8192, 8192), ("tc_bf16_2sm_w", 32768, 32768, 32768), ("tc_bf16_2sm_w", 65536, 256, 4096),
             ("tc_tf32_2sm_w", 8192, 8192, 8192), ("tc_bf16_2sm", 8192, 8192, 8192), ("tc_bf16_2sm", 32768, 32768, 32768), ("tc_tf32_2sm", 8192, 8192, 8192),
             ("tc_bf16_2sm", 65536, 256, 4096), ("tc_bf16_2sm", 4096, 4096, 4096), ("tc_bf16_2sm", 1024, 1024, 1024),
             ("tc_bf16", 8192, 8192, 8192), ("tc_bf16", 8192, 8192, 8192, 1), ("tc_tf32", 8192, 8192, 8192),
             ("tc_bf16", 65536, 256, 4096), ("tc_bf16", 4096, 4096, 4096), ("tma_f32", 4096, 4096, 4096),
             ("simt_f32", 4096, 4096, 4096), ("tma_f32", 1024, 1024, 1024), ("simt_f32", 1024, 1024, 1024),
             ("tc_tf32", 1024, 1024, 1024), ("simt_f32", 64, 64, 64), ("tma_f32", 64, 64, 64),
             ("tc_tf32", 64, 64, 64), ("tc_bf16", 32768, 32768, 32768)]
    if len(sys.argv) > 1:   # name:m:n:k[:transB],...
        cases = [tuple(x.split(":")[:1] + [int(v) for v in x.split(":")[1:]]) for x in sys.argv[1].split(",")]
    for c in cases:
        name, m, n, k = c[:4]
        tb = c[4] if len(c) > 4 else 0
        try:
            med, tf = time_variant(ctx, name, m, n, k, transB=tb)
            print(f"{name:9s} {m}x{n}x{k} transB={tb}: {med/1e3:9.1f} us  {tf:8.1f} TFLOP/s", flush=True)
        except Exception as e:  # noqa: BLE001
            print(f"{name} {m}x{n}x{k}: FAILED {e}", flush=True)
        torch.cuda.empty_cache()
    ctx.terminate()
