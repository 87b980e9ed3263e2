"""BASELINE config 3: 8192^3 GEMM on one B200 (BF16 and TF32 tcgen05 variants).

For each precision class: train the history selector on the key (calibration), then time every
eligible variant exhaustively (burst: best and median of R launches after warm-up; sustained: back
to back for `secs` seconds with the SM clock sampled), and torch.matmul (cuBLAS) as a yardstick.
Target (BASELINE.json north_star): a tcgen05 variant >= 70 % of the measured dense BF16 peak
(MEASURED_PEAKS.json bf16_tflops, burst) at 8192^3; selector within 5 % of the best variant.

    python tools/config3.py [out.json] [secs]
"""
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import gen  # noqa: E402
from bench import ClockSampler, fair_medians, load_peaks  # noqa: E402
from gen.device import device_matrix  # noqa: E402
from paper_2311_03543_b200 import compar as cm  # noqa: E402

R = 10
S = 8192


def burst(run, R=R):
    for _ in range(3):
        run()
    ns = [run() for _ in range(R)]
    return min(ns), statistics.median(ns)


def sustained(fn, flops, secs):
    fn()
    torch.cuda.synchronize()
    clk = ClockSampler(torch.cuda.current_device())
    clk.start()
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
    c = clk.stop()
    return {"tflops": flops * n / (e0.elapsed_time(e1) * 1e-3) / 1e12, "sm_mhz": c.get("sm_mhz"),
            "reasons": c.get("reasons"), "power_w_max": c.get("power_w_max"), "launches": n}


def main(out_path, secs):
    torch.cuda.set_device(0)
    peaks, src = load_peaks()
    ctx = cm.Compar()
    names = [n for n, _ in ctx.variants()]
    flops = 2.0 * S ** 3
    res = {"shape": [S, S, S], "alpha": 1.5, "R": R, "peaks": peaks, "peak_source": src, "cases": []}
    for dt, compute, targets, peak in (("bf16", cm.COMPUTE_BF16, cm.TARGETS_BF16, peaks["bf16_tflops"]),
                                       ("f32", cm.COMPUTE_TF32, cm.TARGETS_TF32, peaks["bf16_tflops"] / 2)):
        A = device_matrix(gen.TAG_A, S, S, dtype=dt)
        B = device_matrix(gen.TAG_B, S, S, dtype=dt)
        C = device_matrix(gen.TAG_C, S, S)
        for beta in (0.5, 0.0):
            ind = cm.BF16 if dt == "bf16" else cm.F32
            mk = lambda hint=-1: cm.make_desc(S, S, S, A=A, B=B, C_in=C, C_out=C, alpha=1.5, beta=beta,  # noqa
                                              in_dtype=ind, compute=compute, variant_hint=hint)
            d = mk()
            calib = 0
            while ctx.select(d)[1] != cm.MODE_MODEL and calib < 64:
                ctx.run(d)
                calib += 1
            sel = [ctx.run(d) for _ in range(R)]
            chosen = sel[-1].variant
            E = [v for v in ctx.eligible(d) if ctx.variants()[v][1] in targets]
            per = {}
            tc = [v for v in E if names[v].startswith("tc_")]
            ffma = [v for v in E if v not in tc]
            # per-variant burst time: bench.fair_medians (idle gap + warm-up before each variant's
            # timed launches, rotated order; median over rounds of the per-round mean)
            descs = {v: mk(v) for v in E}
            fm = fair_medians(ctx, {v: descs[v] for v in tc}, rounds=5, per_round=3)
            for v in tc:
                m = fm[v]
                per[names[v]] = {"median_ns": m, "tflops_median": flops / m / 1e3,
                                 "frac_median": flops / m / 1e3 / peak}
            for v in ffma:   # FFMA variants: 10-50x slower here, 3 launches are enough for the regret
                b, m = burst(lambda: ctx.run(descs[v]).ns, R=3)
                per[names[v]] = {"best_ns": b, "median_ns": m, "tflops_median": flops / m / 1e3}
            if secs > 0:     # sustained, after all bursts; 1 s idle before each
                for v in tc:
                    time.sleep(1.0)
                    per[names[v]]["sustained"] = sustained(lambda: ctx.submit(descs[v]), flops, secs)
                    ctx.sync()
            best = min(per, key=lambda n: per[n]["median_ns"])
            case = {"dtype": dt, "compute": compute, "beta": beta, "peak_tflops": peak,
                    "calibration_runs": calib, "chosen": names[chosen], "best": best,
                    "regret": per[names[chosen]]["median_ns"] / per[best]["median_ns"] - 1.0,
                    "selected_median_tflops": flops / statistics.median(r.ns for r in sel) / 1e3,
                    "variants": per}
            # cuBLAS yardstick (torch.matmul; BF16 -> BF16 out, TF32 via allow_tf32), burst + sustained
            if beta == 0.5:
                torch.backends.cuda.matmul.allow_tf32 = True
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

                def mm():
                    e0.record()
                    torch.matmul(A, B)
                    e1.record()
                    torch.cuda.synchronize()
                    return int(e0.elapsed_time(e1) * 1e6)
                time.sleep(1.0)
                b, m = burst(mm)
                case["cublas"] = {"best_ns": b, "median_ns": m, "tflops_best": flops / b / 1e3,
                                  "tflops_median": flops / m / 1e3}
                if secs > 0:
                    time.sleep(1.0)
                    case["cublas"]["sustained"] = sustained(lambda: torch.matmul(A, B), flops, secs)
                # the same operation through cuBLAS: C_out = 1.5 AB + 0.5 C_in, FP32 C in and out
                # (BF16 inputs: addmm with out_dtype=float32; F32 inputs: TF32 addmm)
                kw = {"out_dtype": torch.float32} if dt == "bf16" else {}

                def mm_same():
                    e0.record()
                    torch.addmm(C, A, B, beta=0.5, alpha=1.5, **kw)
                    e1.record()
                    torch.cuda.synchronize()
                    return int(e0.elapsed_time(e1) * 1e6)
                time.sleep(1.0)
                b, m = burst(mm_same)
                case["cublas_same_op"] = {"best_ns": b, "median_ns": m, "tflops_best": flops / b / 1e3,
                                          "tflops_median": flops / m / 1e3}
                if secs > 0:
                    time.sleep(1.0)
                    case["cublas_same_op"]["sustained"] = sustained(
                        lambda: torch.addmm(C, A, B, beta=0.5, alpha=1.5, **kw), flops, secs)
            res["cases"].append(case)
            print(json.dumps({k: v for k, v in case.items() if k != "variants"}), flush=True)
            for n, p in per.items():
                print("   ", n, json.dumps(p), flush=True)
        del A, B, C
        torch.cuda.empty_cache()
    ctx.terminate()
    with open(out_path, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/config3.json",
         float(sys.argv[2]) if len(sys.argv) > 2 else 2.0)
