"""Calibration-pruning threshold sweep (R32) on the config-5b mixed stream: for each
prune percentage, the history scheduler's stream span over the sum of per-shape best and its
per-shape regret.  Development aid: python tools/prune_sweep.py [pct ...]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import numpy as np  # noqa: E402

import selector_sweep as ss  # noqa: E402
from paper_2311_03543_b200 import compar as cm  # noqa: E402

pcts = [int(x) for x in sys.argv[1:]] or [300, 200, 150, 125]
shapes = [(64, 64, 64), (256, 256, 256), (1024, 1024, 1024), (4096, 4096, 4096), (8192, 8192, 8192),
          (65536, 256, 4096), (4096, 4096, 256)]
rng = np.random.Generator(np.random.PCG64(7))
stream = [shapes[i] for i in rng.integers(0, len(shapes), 200)]
probs = {s: ss.Problem(*s, beta=0.0) for s in shapes}
ctxb = cm.Compar()
names = [n for n, _ in ctxb.variants()]
best = {}
for s, p in probs.items():
    med = ss.exhaustive(ctxb, p, cm.COMPUTE_TF32, ss.eligible(ctxb, ss.TF32_T, p, cm.COMPUTE_TF32))
    best[s] = (min(med, key=med.get), min(med.values()), {names[v]: x for v, x in med.items()})
ctxb.terminate()
sob = sum(best[s][1] for s in stream) / 1e6
for pct in pcts:
    c = cm.Compar(sched=0, calib_prune=pct)
    chosen, span = [], 0
    for s in stream:
        r = c.run(probs[s].desc(cm.COMPUTE_TF32))
        chosen.append((s, r.variant, r.mode))
        span += r.total_ns
    c.terminate()
    calib = sum(1 for (_, _, md) in chosen if md in (cm.MODE_WARMUP, cm.MODE_CALIB))
    reg = {}
    for s in shapes:
        vs = [v for (ss_, v, md) in chosen if ss_ == s and md == cm.MODE_MODEL]
        if vs:
            v = max(set(vs), key=vs.count)
            reg[str(list(s))] = round(best[s][2][names[v]] / best[s][1] - 1.0, 4)
    print(json.dumps({"prune_pct": pct, "span_ms": span / 1e6, "sum_of_best_ms": sob, "span_over_best": span / 1e6 / sob,
                      "calibration_runs": calib, "max_regret": max(reg.values()), "regret": reg}), flush=True)
