"""Kernel-only times (ncu gpu__time_duration) of the single-wave tensor-core shapes: every tcgen05
variant / tile-width knob and cuBLAS on the same operation (FP32 C in and out), 5 launches each,
groups separated by a one-element torch kernel.

  ncu --metrics gpu__time_duration.sum --csv --log-file OUT.csv python tools/single_wave_ncu.py run
  python tools/single_wave_ncu.py parse OUT.csv [out.json]
"""
import csv
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SHAPES = [(1024, "bf16"), (2048, "bf16"), (1024, "f32"), (2048, "f32")]
CONFIGS = [("tc", "COMPAR_TC1_BN", "256"), ("tc", "COMPAR_TC1_BN", "128"), ("tc", "COMPAR_TC1_BN", "64"),
           ("tc2", "COMPAR_TC2_BN", "256"), ("tc2", "COMPAR_TC2_BN", "128"), ("w", None, None), ("ck", None, None),
           ("cublas", None, None)]
REPS = 5


def labels():
    out = []
    for s, dt in SHAPES:
        pre = "tc_bf16" if dt == "bf16" else "tc_tf32"
        for fam, env, val in CONFIGS:
            name = {"tc": pre, "tc2": pre + "_2sm", "w": pre + "_2sm_w", "ck": pre + "_ck",
                    "cublas": "cublas_addmm_f32out"}[fam]
            out.append(f"{s}^3_{dt}/{name}{'/' + val if val else ''}")
    return out


def run():
    import torch

    import gen
    from gen.device import device_matrix
    from paper_2311_03543_b200 import compar as cm
    torch.cuda.set_device(0)
    mark = torch.zeros(1, device="cuda")
    for s, dt in SHAPES:
        A = device_matrix(gen.TAG_A, s, s, dtype=dt)
        B = device_matrix(gen.TAG_B, s, s, dtype=dt)
        C = device_matrix(gen.TAG_C, s, s)
        pre = "tc_bf16" if dt == "bf16" else "tc_tf32"
        for fam, env, val in CONFIGS:
            mark.add_(1)
            if fam == "cublas":
                torch.backends.cuda.matmul.allow_tf32 = dt == "f32"
                out = torch.empty_like(C)
                kw = dict(beta=0.5, alpha=1.5, out=out)
                if dt == "bf16":
                    kw["out_dtype"] = torch.float32
                for _ in range(REPS):
                    torch.addmm(C, A, B, **kw)
                continue
            if env:
                os.environ[env] = val
            ctx = cm.Compar()
            if env:
                os.environ.pop(env)
            names = [v for v, _ in ctx.variants()]
            name = {"tc": pre, "tc2": pre + "_2sm", "w": pre + "_2sm_w", "ck": pre + "_ck"}[fam]
            d = cm.make_desc(s, s, s, A=A, B=B, C_in=C, C_out=C, alpha=1.5, beta=0.5,
                             in_dtype=cm.BF16 if dt == "bf16" else cm.F32,
                             compute=cm.COMPUTE_BF16 if dt == "bf16" else cm.COMPUTE_TF32,
                             variant_hint=names.index(name), stream=torch.cuda.current_stream().cuda_stream)
            for _ in range(REPS):
                ctx.run(d)
            ctx.terminate()
    mark.add_(1)
    torch.cuda.synchronize()


def parse(path, out=None):
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    for r in csv.DictReader(lines):
        if r.get("Metric Name") == "gpu__time_duration.sum" and "fill_kernel" not in r["Kernel Name"] \
                and "FillFunctor" not in r["Kernel Name"]:
            rows.append((r["Kernel Name"], float(r["Metric Value"]) * scale[r["Metric Unit"]]))
    groups, cur = [], None
    for name, us in rows:
        if "CUDAFunctorOnSelf_add" in name:         # the separator (mark.add_(1))
            if cur is not None:
                groups.append(cur)
            cur = []
        elif cur is not None:
            cur.append((name, us))
    res = {}
    for lab, g in zip(labels(), groups):
        # cuBLAS may launch more than one kernel per call: sum per call
        per = len(g) // REPS if g else 1
        calls = [sum(u for _, u in g[i * per:(i + 1) * per]) for i in range(REPS)] if g else []
        res[lab] = {"median_us": statistics.median(calls) if calls else None,
                    "kernels": sorted({n[:60] for n, _ in g})}
        print(f"{lab:45s} {res[lab]['median_us']:8.2f} us  {res[lab]['kernels']}")
    if out:
        with open(out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run()
    else:
        parse(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
