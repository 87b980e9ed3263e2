"""Yardstick for the strict-FP32 class: tma_f32 against cuBLAS SGEMM on the same operation
(torch.addmm with TF32 disabled: C = 1.5 A B + 0.5 C, FP32 in / out), interleaved, medians of
event-timed launches.  Development aid.

  python tools/sgemm_yardstick.py [n ...]
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

torch.backends.cuda.matmul.allow_tf32 = False
torch.backends.cuda.matmul.allow_fp16_reduced_precision_reduction = False
ctx = cm.Compar()
names = [v for v, _ in ctx.variants()]
for n in [int(x) for x in sys.argv[1:]] or [2048, 4096, 8192]:
    A = device_matrix(gen.TAG_A, n, n)
    B = device_matrix(gen.TAG_B, n, n)
    C = device_matrix(gen.TAG_C, n, n)
    d = cm.make_desc(n, n, n, A=A, B=B, C_in=C, C_out=C, alpha=1.5, beta=0.5, compute=cm.COMPUTE_F32_STRICT,
                     variant_hint=names.index("tma_f32"), stream=torch.cuda.current_stream().cuda_stream)
    ours, cub = [], []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for r in range(12):
        ctx.run(d)
        torch.cuda.synchronize()
        ours.append(ctx.run(d).ns / 1e3)
        torch.addmm(C, A, B, beta=0.5, alpha=1.5, out=C)
        torch.cuda.synchronize()
        e0.record()
        torch.addmm(C, A, B, beta=0.5, alpha=1.5, out=C)
        e1.record()
        torch.cuda.synchronize()
        cub.append(e0.elapsed_time(e1) * 1e3)
    fl = 2.0 * n ** 3
    o, c = statistics.median(ours[2:]), statistics.median(cub[2:])
    print({"n": n, "tma_f32_us": round(o, 1), "tma_f32_tflops": round(fl / o / 1e6, 2),
           "cublas_sgemm_us": round(c, 1), "cublas_tflops": round(fl / c / 1e6, 2), "ours_over_cublas": round(c / o, 3)})
