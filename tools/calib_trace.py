"""Calibration-order diagnostic at the bench workload (32768^3 BF16 by default).

Prints per-execution kernel ns for (1) the selector's own calibration + model trace and (2) hinted
executions in interleaved order (v0 v1 v2 v3 v0 ...) and in blocked order (v0 x4, v1 x4, ...), to
show how the preceding kernel's power draw biases a sample on the power-capped B200.
usage: python tools/calib_trace.py [size] [out.json]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import gen  # noqa: E402
from gen.device import device_matrix  # noqa: E402
from paper_2311_03543_b200 import compar as cm  # noqa: E402


def main():
    s = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
    out = sys.argv[2] if len(sys.argv) > 2 else None
    torch.cuda.set_device(0)
    A = device_matrix(gen.TAG_A, s, s, dtype="bf16")
    B = device_matrix(gen.TAG_B, s, s, dtype="bf16")
    C = device_matrix(gen.TAG_C, s, s)
    res = {}
    for order in ("blocked", "interleaved"):
        os.environ["COMPAR_CALIB_ORDER"] = order
        ctx = cm.Compar()
        names = [n for n, _ in ctx.variants()]
        d = cm.make_desc(s, s, s, A=A, B=B, C_in=C, C_out=C, alpha=1.5, beta=0.5, in_dtype=cm.BF16,
                         compute=cm.COMPUTE_BF16)
        tr = []
        for _ in range(40):
            r = ctx.run(d)
            tr.append([names[r.variant], r.mode, r.ns])
        res[f"selector_{order}"] = tr
        ctx.terminate()
    os.environ.pop("COMPAR_CALIB_ORDER", None)
    ctx = cm.Compar()
    names = [n for n, _ in ctx.variants()]
    E = ctx.eligible(cm.make_desc(s, s, s, A=A, B=B, C_in=C, C_out=C, alpha=1.5, beta=0.5, in_dtype=cm.BF16,
                                  compute=cm.COMPUTE_BF16))

    def hinted(seq):
        tr = []
        for v in seq:
            d = cm.make_desc(s, s, s, A=A, B=B, C_in=C, C_out=C, alpha=1.5, beta=0.5, in_dtype=cm.BF16,
                             compute=cm.COMPUTE_BF16, variant_hint=v)
            tr.append([names[v], ctx.run(d).ns])
        return tr

    res["hint_interleaved"] = hinted(E * 4)
    res["hint_blocked"] = hinted([v for v in E for _ in range(4)])
    tc = [v for v in E if names[v] != "simt_bf16"]
    res["hint_interleaved_tc_only"] = hinted(tc * 4)
    txt = json.dumps(res, indent=0)
    if out:
        with open(out, "w") as f:
            f.write(txt)
    for k, tr in res.items():
        print(k)
        for row in tr:
            print("   ", *row)


if __name__ == "__main__":
    main()
