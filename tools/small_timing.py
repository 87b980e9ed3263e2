"""Are small-GEMM event timings inflated by idle clocks / host gaps?  Compare per-task ns when
tasks are synced one by one vs submitted back to back (GPU kept busy)."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import gen  # noqa: E402
from gen.device import device_matrix  # noqa: E402
from paper_2311_03543_b200 import compar as cm  # noqa: E402

ctx = cm.Compar()
names = [v for v, _ in ctx.variants()]
for s in (64, 256, 1024):
    A = device_matrix(gen.TAG_A, s, s)
    B = device_matrix(gen.TAG_B, s, s)
    Cd = device_matrix(gen.TAG_C, s, s)
    for v in ("simt_f32", "tma_f32", "tc_tf32", "tc_tf32_2sm"):
        d = cm.make_desc(s, s, s, A=A, B=B, C_in=Cd, C_out=Cd, alpha=1.0, beta=0.0, compute=cm.COMPUTE_TF32,
                         variant_hint=names.index(v))
        one = [ctx.run(d).ns for _ in range(30)]
        tids = [ctx.submit(d) for _ in range(30)]
        many = [ctx.sync(t).ns for t in tids]
        # long busy loop of the same kernel timed as a batch with torch events
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        tids = [ctx.submit(d) for _ in range(200)]
        e1.record()
        ctx.sync()
        torch.cuda.synchronize()
        batch = e0.elapsed_time(e1) * 1e6 / 200
        print(f"{s}^3 {v:12s} synced-one-by-one median {statistics.median(one)/1e3:7.1f} us | back-to-back "
              f"median {statistics.median(many)/1e3:7.1f} us | batch avg {batch/1e3:7.1f} us", flush=True)
        # cuBLAS beside (torch.addmm, TF32), same batch protocol
    torch.backends.cuda.matmul.allow_tf32 = True
    for _ in range(3):
        torch.addmm(Cd, A, B)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(200):
        torch.addmm(Cd, A, B)
    e1.record()
    torch.cuda.synchronize()
    print(f"{s}^3 cublas addmm batch avg {e0.elapsed_time(e1) * 1e3 / 200:7.1f} us", flush=True)
x = torch.zeros(1, device="cuda")
torch.cuda.synchronize()
e0.record()
for _ in range(200):
    x.add_(1)
e1.record()
torch.cuda.synchronize()
print(f"one-element torch kernel (launch floor) batch avg {e0.elapsed_time(e1) * 1e3 / 200:7.2f} us", flush=True)
ctx.terminate()
