"""Run one variant at one shape `reps` times (target for ncu captures / quick timing).

usage: python tools/prof_run.py NAME M N K [reps] [transB] [--pad P] [--beta B]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import gen  # noqa: E402
from gen.device import device_matrix  # noqa: E402
from paper_2311_03543_b200 import compar as cm  # noqa: E402

if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("name")
    ap.add_argument("m", type=int)
    ap.add_argument("n", type=int)
    ap.add_argument("k", type=int)
    ap.add_argument("reps", type=int, nargs="?", default=3)
    ap.add_argument("transB", type=int, nargs="?", default=0)
    ap.add_argument("--pad", type=int, default=0, help="extra elements on every leading dimension")
    ap.add_argument("--beta", type=float, default=0.5)
    a = ap.parse_args()
    name, m, n, k, tb = a.name, a.m, a.n, a.k, a.transB
    ctx = cm.Compar()
    names = [v for v, _ in ctx.variants()]
    bf = "bf16" in name
    dt = "bf16" if bf else "f32"
    lda = k + a.pad
    ldb = (k if tb else n) + a.pad
    ldc = n + a.pad
    A = device_matrix(gen.TAG_A, m, k, dtype=dt, ld=lda)
    B = device_matrix(gen.TAG_B, k, n, dtype=dt, transposed=bool(tb), ld=ldb)
    Cd = device_matrix(gen.TAG_C, m, n, ld=ldc)
    compute = cm.COMPUTE_BF16 if bf else (cm.COMPUTE_TF32 if "tf32" in name else
                                          cm.COMPUTE_F32_SPLIT if name == "tc_f32x3" else cm.COMPUTE_F32_STRICT)
    d = cm.make_desc(m, n, k, A=A.data_ptr(), B=B.data_ptr(), C_in=Cd.data_ptr(), C_out=Cd.data_ptr(), lda=lda,
                     ldb=ldb, ldc_in=ldc, ldc_out=ldc, alpha=1.5, beta=a.beta, in_dtype=cm.BF16 if bf else cm.F32,
                     compute=compute, transB=tb, variant_hint=names.index(name))
    for _ in range(a.reps):
        r = ctx.run(d)
        print(f"{name} {m}x{n}x{k} pad={a.pad} beta={a.beta}: {r.ns / 1e3:.1f} us  "
              f"{2.0 * m * n * k / r.ns / 1e3:.1f} TFLOP/s", flush=True)
    ctx.terminate()
