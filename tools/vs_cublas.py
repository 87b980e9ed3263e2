"""Yardstick: our tcgen05 variants vs torch.matmul (cuBLAS, the MEASURED_PEAKS reference) under
the same thermal/power conditions, back to back for ~`secs` seconds each (sustained)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import gen  # noqa: E402
from gen.device import device_matrix  # noqa: E402
from paper_2311_03543_b200 import compar as cm  # noqa: E402


def sustained(fn, flops, secs):
    from bench import ClockSampler
    fn()
    torch.cuda.synchronize()
    clk = ClockSampler(torch.cuda.current_device())
    clk.start()
    tf = _sustained(fn, flops, secs)
    c = clk.stop()
    mhz = c.get("sm_mhz") or float("nan")
    return f"{tf:.0f}TF@{mhz:.0f}MHz({tf / (148 * 8192 * mhz * 1e-6):.0%}/clk,{c.get('power_w_max')}W)"


def _sustained(fn, flops, secs):
    n, t0 = 0, time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    while time.perf_counter() - t0 < secs:
        fn()
        n += 1
        if n % 8 == 0:
            torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    return flops * n / (e0.elapsed_time(e1) * 1e-3) / 1e12


if __name__ == "__main__":
    secs = float(sys.argv[1]) if len(sys.argv) > 1 else 3.0
    ctx = cm.Compar()
    names = [v for v, _ in ctx.variants()]
    for s in [int(x) for x in (sys.argv[2].split(',') if len(sys.argv) > 2 else (8192, 16384, 32768))]:
        A = device_matrix(gen.TAG_A, s, s, dtype="bf16")
        B = device_matrix(gen.TAG_B, s, s, dtype="bf16")
        Cd = device_matrix(gen.TAG_C, s, s)
        flops = 2.0 * s ** 3
        res = {}
        for v in ("tc_bf16", "tc_bf16_2sm", "tc_bf16_2sm_w"):
            d = cm.make_desc(s, s, s, A=A, B=B, C_in=Cd, C_out=Cd, alpha=1.5, beta=0.5, in_dtype=cm.BF16,
                             compute=cm.COMPUTE_BF16, variant_hint=names.index(v))
            res[v] = sustained(lambda: ctx.submit(d), flops, secs)
            ctx.sync()
        d0 = cm.make_desc(s, s, s, A=A, B=B, C_in=Cd, C_out=Cd, alpha=1.0, beta=0.0, in_dtype=cm.BF16,
                          compute=cm.COMPUTE_BF16, variant_hint=names.index("tc_bf16_2sm"))
        res["tc_bf16_2sm(beta=0)"] = sustained(lambda: ctx.submit(d0), flops, secs)
        ctx.sync()
        out = torch.empty((s, s), dtype=torch.bfloat16, device="cuda")
        res["torch.matmul(bf16->bf16)"] = sustained(lambda: torch.matmul(A, B, out=out), flops, secs)
        del out
        # the same operation as ours: C = 1.5 AB + 0.5 C, FP32 C in and out
        out = torch.empty((s, s), dtype=torch.float32, device="cuda")
        res["torch.addmm(same op, f32 C)"] = sustained(
            lambda: torch.addmm(Cd, A, B, beta=0.5, alpha=1.5, out_dtype=torch.float32, out=out), flops, secs)
        print(f"{s}^3 sustained {secs:.0f}s: " + "  ".join(f"{k}={v}" for k, v in res.items()), flush=True)
        del A, B, Cd, out
        torch.cuda.empty_cache()
    ctx.terminate()
