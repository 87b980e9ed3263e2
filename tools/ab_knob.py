"""A/B of a launcher knob (read at compar_init) on one variant: per shape, alternating rounds of
knob=A / knob=B, each a fresh context; median per-task event time over 10 synced runs after 2
warm-ups, and the back-to-back time of 10 submits.  Development aid.

  python tools/ab_knob.py VARIANT ENV VAL_A VAL_B DTYPE(f32|bf16) COMPUTE(strict|tf32|bf16|split) M N K [M N K ...]
"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import gen  # noqa: E402
from gen.device import device_matrix  # noqa: E402
from paper_2311_03543_b200 import compar as cm  # noqa: E402

var, env, va, vb, dt, comp = sys.argv[1:7]
dims = [int(x) for x in sys.argv[7:]]
compute = {"strict": cm.COMPUTE_F32_STRICT, "tf32": cm.COMPUTE_TF32, "bf16": cm.COMPUTE_BF16,
           "split": cm.COMPUTE_F32_SPLIT}[comp]
for i in range(0, len(dims), 3):
    m, n, k = dims[i:i + 3]
    A = device_matrix(gen.TAG_A, m, k, dtype=dt)
    B = device_matrix(gen.TAG_B, k, n, dtype=dt)
    C0 = device_matrix(gen.TAG_C, m, n)
    res = {va: [], vb: []}
    outs = {}
    for rnd in range(3):
        for val in (va, vb) if rnd % 2 == 0 else (vb, va):
            os.environ[env] = val
            ctx = cm.Compar()
            os.environ.pop(env)
            names = [v for v, _ in ctx.variants()]
            C = C0.clone()
            d = cm.make_desc(m, n, k, A=A, B=B, C_in=C, C_out=C, alpha=1.5, beta=0.5,
                             in_dtype=cm.BF16 if dt == "bf16" else cm.F32, compute=compute,
                             variant_hint=names.index(var), stream=torch.cuda.current_stream().cuda_stream)
            for _ in range(2):
                ctx.run(d)
            ns = [ctx.run(d).ns for _ in range(10)]
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ids = [ctx.submit(d) for _ in range(10)]
            e1.record()
            torch.cuda.synchronize()
            for t in ids:
                ctx.sync(t)
            res[val].append((statistics.median(ns) / 1e3, e0.elapsed_time(e1) * 100.0))
            C2 = C0.clone()
            d2 = cm.make_desc(m, n, k, A=A, B=B, C_in=C2, C_out=C2, alpha=1.5, beta=0.5,
                              in_dtype=cm.BF16 if dt == "bf16" else cm.F32, compute=compute,
                              variant_hint=names.index(var), stream=torch.cuda.current_stream().cuda_stream)
            ctx.run(d2)
            outs[val] = C2
            ctx.terminate()
    same = torch.equal(outs[va], outs[vb])
    fl = 2.0 * m * n * k
    for val in (va, vb):
        t = [x[0] for x in res[val]]
        b = [x[1] for x in res[val]]
        print(f"{var} {m}x{n}x{k} {env}={val}: task us {[round(x, 1) for x in t]} "
              f"({fl / statistics.median(t) / 1e6:.1f} TFLOP/s) | b2b us {[round(x, 1) for x in b]} | bitwise_equal={same}")
