"""Single-wave tensor-core shapes: every tcgen05 variant and tile-width knob
against cuBLAS on the same operation, at 1024^3 / 2048^3 (BF16 and TF32), beta = 0.5.

Two timings per configuration, both per launch:
  * task: median of the runtime's own per-task event sample over 40 synced runs (what the
    selector sees);
  * b2b:  200 launches back to back through the runtime, torch events around the batch.
cuBLAS: torch.addmm(C, A, B, beta=0.5, alpha=1.5, out_dtype=float32) — FP32 C in and out.
usage: python tools/single_wave.py [out.json]
"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import gen  # noqa: E402
from gen.device import device_matrix  # noqa: E402
from paper_2311_03543_b200 import compar as cm  # noqa: E402

KNOBS = {"tc": ("COMPAR_TC1_BN", ["256", "128", "64"]), "tc2": ("COMPAR_TC2_BN", ["256", "128"]), "w": (None, [None])}


def time_cfg(variant, env, val, m, n, k, dt, A, B, C):
    if env:
        os.environ[env] = val
    try:
        ctx = cm.Compar()
    finally:
        if env:
            os.environ.pop(env, None)
    names = [v for v, _ in ctx.variants()]
    d = cm.make_desc(m, n, k, A=A, B=B, C_in=C, C_out=C, alpha=1.5, beta=0.5,
                     in_dtype=cm.BF16 if dt == "bf16" else cm.F32,
                     compute=cm.COMPUTE_BF16 if dt == "bf16" else cm.COMPUTE_TF32,
                     variant_hint=names.index(variant), stream=torch.cuda.current_stream().cuda_stream)
    for _ in range(5):
        ctx.run(d)
    task = statistics.median(ctx.run(d).ns for _ in range(40)) / 1e3
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    ts = [ctx.submit(d) for _ in range(200)]
    e1.record()
    ctx.sync()
    torch.cuda.synchronize()
    b2b = e0.elapsed_time(e1) * 1e3 / 200
    ctx.terminate()
    return task, b2b


def cublas(A, B, C, dt):
    torch.backends.cuda.matmul.allow_tf32 = dt == "f32"
    out = torch.empty_like(C)
    kw = dict(beta=0.5, alpha=1.5, out=out)
    if dt == "bf16":
        kw["out_dtype"] = torch.float32
    for _ in range(5):
        torch.addmm(C, A, B, **kw)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    one = []
    for _ in range(40):
        torch.cuda.synchronize()
        e0.record()
        torch.addmm(C, A, B, **kw)
        e1.record()
        torch.cuda.synchronize()
        one.append(e0.elapsed_time(e1) * 1e3)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(200):
        torch.addmm(C, A, B, **kw)
    e1.record()
    torch.cuda.synchronize()
    return statistics.median(one), e0.elapsed_time(e1) * 1e3 / 200


def main(out_path):
    torch.cuda.set_device(0)
    res = {}
    for s in (1024, 2048):
        for dt in ("bf16", "f32"):
            A = device_matrix(gen.TAG_A, s, s, dtype=dt)
            B = device_matrix(gen.TAG_B, s, s, dtype=dt)
            C = device_matrix(gen.TAG_C, s, s)
            key = f"{s}^3_{dt}"
            row = {}
            pre = "tc_bf16" if dt == "bf16" else "tc_tf32"
            for fam, (env, vals) in KNOBS.items():
                variant = {"tc": pre, "tc2": pre + "_2sm", "w": pre + "_2sm_w"}[fam]
                for v in vals:
                    task, b2b = time_cfg(variant, env, v, s, s, s, dt, A, B, C)
                    row[f"{variant}{'/' + v if v else ''}"] = {"task_us": task, "b2b_us": b2b}
                    print(key, variant, v, f"task {task:.2f} us  b2b {b2b:.2f} us", flush=True)
            one, b2b = cublas(A, B, C, dt)
            row["cublas_addmm_f32out"] = {"task_us": one, "b2b_us": b2b}
            print(key, "cublas", f"single {one:.2f} us  b2b {b2b:.2f} us", flush=True)
            res[key] = row
    if out_path:
        with open(out_path, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else None)
