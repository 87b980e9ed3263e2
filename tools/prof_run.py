"""Run one variant at one shape `reps` times (target for ncu captures).

usage: python tools/prof_run.py NAME M N K [reps] [transB]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import gen  # noqa: E402
from gen.device import device_matrix  # noqa: E402
from paper_2311_03543_b200 import compar as cm  # noqa: E402

if __name__ == "__main__":
    name, m, n, k = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
    reps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
    tb = int(sys.argv[6]) if len(sys.argv) > 6 else 0
    ctx = cm.Compar()
    names = [v for v, _ in ctx.variants()]
    bf = "bf16" in name
    dt = "bf16" if bf else "f32"
    A = device_matrix(gen.TAG_A, m, k, dtype=dt)
    B = device_matrix(gen.TAG_B, k, n, dtype=dt, transposed=bool(tb))
    Cd = device_matrix(gen.TAG_C, m, n)
    compute = cm.COMPUTE_BF16 if bf else (cm.COMPUTE_TF32 if "tf32" in name else cm.COMPUTE_F32_STRICT)
    d = cm.make_desc(m, n, k, A=A, B=B, C_in=Cd, C_out=Cd, alpha=1.5, beta=0.5, in_dtype=cm.BF16 if bf else cm.F32,
                     compute=compute, transB=tb, ldb=(k if tb else n), variant_hint=names.index(name))
    for _ in range(reps):
        r = ctx.run(d)
        print(f"{name} {m}x{n}x{k}: {r.ns / 1e3:.1f} us  {2.0 * m * n * k / r.ns / 1e3:.1f} TFLOP/s", flush=True)
    ctx.terminate()
