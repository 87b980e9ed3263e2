"""Host-side cost of the ABI calls (the paper's 'decision overhead'): wall time of
compar_gemm_submit and compar_sync for a tiny task, with a variant hint and with the selector in
model mode, plus the raw ctypes round trip of a no-op ABI call."""
import ctypes
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import gen  # noqa: E402
from gen.device import device_matrix  # noqa: E402
from paper_2311_03543_b200 import compar as cm  # noqa: E402

ctx = cm.Compar()
names = [v for v, _ in ctx.variants()]
A = device_matrix(gen.TAG_A, 64, 64)
B = device_matrix(gen.TAG_B, 64, 64)
Cd = device_matrix(gen.TAG_C, 64, 64)
torch.cuda.synchronize()
st = cm.Stats()
t = []
for _ in range(2000):
    t0 = time.perf_counter()
    cm.lib.compar_stats_get(ctx.ctx, ctypes.byref(st))
    t.append(time.perf_counter() - t0)
print(f"ctypes no-op ABI call: {statistics.median(t) * 1e6:.2f} us")
cases = [("hint " + v, names.index(v)) for v in ("simt_f32", "tma_f32", "tc_tf32", "tc_tf32_2sm", "tc_tf32_2sm_w")]
for label, hint in cases + [("selector (model mode)", -1)]:
    d = cm.make_desc(64, 64, 64, A=A, B=B, C_in=Cd, C_out=Cd, alpha=1.0, beta=0.0, compute=cm.COMPUTE_TF32,
                     variant_hint=hint)
    for _ in range(40):
        ctx.run(d)
    sub, syn = [], []
    for _ in range(500):
        t0 = time.perf_counter()
        task = ctx.submit(d)
        t1 = time.perf_counter()
        ctx.sync(task)
        t2 = time.perf_counter()
        sub.append(t1 - t0)
        syn.append(t2 - t1)
    print(f"{label}: submit {statistics.median(sub) * 1e6:.2f} us, sync (incl. GPU wait) "
          f"{statistics.median(syn) * 1e6:.2f} us", flush=True)
ctx.terminate()
