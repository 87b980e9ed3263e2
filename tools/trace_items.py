"""Per-item timeline of the CTA-pair kernel (tc_gemm_2sm_mc) on one shape: for every CTA (< 160)
and work item (< 8), globaltimer stamps of the item's first TMA, its accumulator commit (leader
CTAs) and its last C_out store.  Development aid (needs the -DCOMPAR_TRACE library:
`python tools/trace_pair.py build`).

  python tools/trace_items.py M N K [beta] [variant]

Prints, per item index j, the spread over CTAs of start / commit / end (µs from the first CTA
entry), plus the CTAs' exit spread: where a launch loses time (ramp, per-wave rate, tail).
"""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["COMPAR_LIB"] = os.environ.get("COMPAR_LIB") or os.path.join(ROOT, "build_trace", "libcompar.so")

import torch  # noqa: E402

import gen  # noqa: E402
from gen.device import device_matrix  # noqa: E402
from paper_2311_03543_b200 import compar as cm  # noqa: E402

m, n, k = (int(x) for x in sys.argv[1:4])
beta = float(sys.argv[4]) if len(sys.argv) > 4 else 0.5
vname = sys.argv[5] if len(sys.argv) > 5 else "tc_bf16_2sm"
lib = ctypes.CDLL(os.environ["COMPAR_LIB"])
ctx = cm.Compar()
names = [v for v, _ in ctx.variants()]
A = device_matrix(gen.TAG_A, m, k, dtype="bf16")
B = device_matrix(gen.TAG_B, k, n, dtype="bf16")
C = device_matrix(gen.TAG_C, m, n)
d = cm.make_desc(m, n, k, A=A, B=B, C_in=C, C_out=C, alpha=1.5, beta=beta, in_dtype=cm.BF16,
                 compute=cm.COMPUTE_BF16, variant_hint=names.index(vname))
buf = (ctypes.c_ulonglong * (160 * 8 * 3))()
cb = (ctypes.c_ulonglong * 320)()
evs = []
for rep_i in range(6):
    assert lib.compar_trace_item_read(buf, 1) == 0
    rep = ctx.run(d)
    evs.append(rep.ns / 1e3)
assert lib.compar_trace_item_read(buf, 0) == 0
assert lib.compar_trace_cta_read(cb) == 0
ctx.terminate()

ent = {i: cb[2 * i] for i in range(160) if cb[2 * i]}
ext = {i: cb[2 * i + 1] for i in range(160) if cb[2 * i + 1]}
e0 = min(ent.values())
us = lambda t: (t - e0) / 1e3  # noqa: E731
out = {"shape": [m, n, k], "beta": beta, "variant": vname, "event_us": evs,
       "entry_spread_us": us(max(ent.values())), "exit_first_us": us(min(ext.values())),
       "exit_last_us": us(max(ext.values())), "items": []}
print(f"{vname} {m}x{n}x{k} beta={beta}: event us {evs[-1]:.1f} (runs {', '.join(f'{e:.1f}' for e in evs)})")
print(f"  ctas {len(ent)}: entry spread {out['entry_spread_us']:.2f} us, exit {out['exit_first_us']:.2f} .. "
      f"{out['exit_last_us']:.2f} us")
for j in range(8):
    rows = []
    for c in range(160):
        s0, s1, s2 = (buf[(c * 8 + j) * 3 + w] for w in range(3))
        if s0 or s2:
            rows.append((c, s0, s1, s2))
    if not rows:
        break
    st = [us(r[1]) for r in rows if r[1]]
    cm_ = [us(r[2]) for r in rows if r[2]]
    en = [us(r[3]) for r in rows if r[3]]
    durs = [(r[3] - r[1]) / 1e3 for r in rows if r[1] and r[3]]
    rec = {"item": j, "ctas": len(rows),
           "start": [min(st), sorted(st)[len(st) // 2], max(st)] if st else None,
           "commit": [min(cm_), sorted(cm_)[len(cm_) // 2], max(cm_)] if cm_ else None,
           "end": [min(en), sorted(en)[len(en) // 2], max(en)] if en else None,
           "dur_median": sorted(durs)[len(durs) // 2] if durs else None}
    out["items"].append(rec)
    f3 = lambda v: "-" if v is None else "/".join(f"{x:6.1f}" for x in v)  # noqa: E731
    print(f"  item {j}: {len(rows):3d} ctas | start {f3(rec['start'])} | commit {f3(rec['commit'])} | "
          f"end {f3(rec['end'])} | start->end median {rec['dur_median'] if rec['dur_median'] is None else round(rec['dur_median'], 1)}")
if len(sys.argv) > 6:
    json.dump(out, open(sys.argv[6], "w"), indent=1)
