"""How much of a task's event time is launch / host latency rather than kernel: per shape, the
runtime's own sample of one task on an idle stream (`rep.ns`, the selector's quantity) against
the per-task time of a back-to-back stream of submits (torch events around 10 submits, one sync:
the host-side prep of task i+1 overlaps kernel i).  Development aid.

  python tools/launch_gap.py [variant] [M N K] ...
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

vname = sys.argv[1] if len(sys.argv) > 1 else "tc_bf16_2sm"
args = [int(x) for x in sys.argv[2:]] or [65536, 256, 4096, 18944, 256, 4096, 2048, 2048, 2048, 256, 256, 64]
ctx = cm.Compar()
names = [v for v, _ in ctx.variants()]
st = torch.cuda.current_stream()
for i in range(0, len(args), 3):
    m, n, k = args[i:i + 3]
    A = device_matrix(gen.TAG_A, m, k, dtype="bf16")
    B = device_matrix(gen.TAG_B, k, n, dtype="bf16")
    C = device_matrix(gen.TAG_C, m, n)
    d = cm.make_desc(m, n, k, A=A, B=B, C_in=C, C_out=C, alpha=1.5, beta=0.5, in_dtype=cm.BF16,
                     compute=cm.COMPUTE_BF16, variant_hint=names.index(vname), stream=st.cuda_stream)
    for _ in range(3):
        ctx.run(d)
    single = statistics.median(ctx.run(d).ns / 1e3 for _ in range(10))
    spans, inner = [], []
    for _ in range(5):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        ids = [ctx.submit(d) for _ in range(10)]
        e1.record(st)
        reps = [ctx.sync(t) for t in ids]
        torch.cuda.synchronize()
        spans.append(e0.elapsed_time(e1) * 1e3 / 10)
        inner.append(statistics.median(r.ns / 1e3 for r in reps[1:]))
    print(f"{vname} {m}x{n}x{k}: idle-stream task {single:.2f} us | back-to-back {statistics.median(spans):.2f} us "
          f"per task (runtime's own per-task events inside the stream {statistics.median(inner):.2f} us)", flush=True)
    del A, B, C
ctx.terminate()
