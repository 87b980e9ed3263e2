"""NEXT-2 on the GPU (-m gpu): the `predict` scheduler (per-variant cost model over shapes,
PAPER.md P:224 / P:308 "additional training of performance models") on a BASELINE config-5b
subset with real kernels and real cudaEvent samples.

* Every decision (variant, mode) equals oracle/selector.py's decide_predict / calibration
  decision (with the R32 pruning and static lower bounds), fed with the runtime's OWN history as
  written by compar_perf_save just before the submit (every task is synced before the next
  decision, so nothing is pending);
* every task's C is checked against the FP64 oracle (small shapes in full; large shapes on
  sampled full rows), at the tolerance of the variant that ran.
"""
import os
import tempfile

import numpy as np
import pytest

import gen
from oracle import gemm as og
from oracle import selector as so

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from gen.device import device_matrix  # noqa: E402
from tests._gpu_util import assert_parity  # noqa: E402

cm = pytest.importorskip("paper_2311_03543_b200.compar")

SHAPES = [(64, 64, 64), (256, 256, 256), (512, 512, 512), (1024, 1024, 1024), (4096, 4096, 256),
          (2048, 2048, 2048), (65536, 256, 4096)]


def load_dump(path, names):
    """Parse compar_perf_save's text format (include/compar.h) into the oracle's history table."""
    hist = {}
    idx = {nm: i for i, nm in enumerate(names)}
    for ln in open(path):
        if not ln.strip() or ln.startswith("#"):
            continue
        f = ln.split()
        if f[0] not in idx:
            continue
        key = tuple(int(x) for x in f[1:8])
        hist[(idx[f[0]], key)] = so.Record(seen=int(f[8]), count=int(f[9]), sum_ns=int(f[10]),
                                           sumsq_ns=int(f[11]), min_ns=int(f[12]))
    return hist


def lb_class(name):
    """R32 arithmetic class of a built-in variant (the static lower bound's peak)."""
    if name.startswith("tc_tf32"):
        return "tf32"
    if name.startswith("tc_bf16"):
        return "bf16"
    if name == "tc_f32x3":
        return "f32x3"
    return "ffma" if name in ("simt_f32", "tma_f32", "simt_bf16") else None


def expected(orc, key, elig, lb):
    """The predict scheduler's decision (runtime compar.cpp choose_core, oracle restatement)."""
    dp = orc.decide_predict(key, elig, lb)
    if dp is not None:
        return dp, orc
    unk = orc.unknown_predict(key, elig, lb)
    if unk and len(unk) < len(elig):
        return orc.decide(key, unk, [lb[elig.index(v)] for v in unk]), orc
    return orc.decide(key, elig, lb), orc


def test_predict_scheduler_real_kernels_match_oracle():
    ctx = cm.Compar(sched=cm.SCHED_PREDICT)
    names = [n for n, _ in ctx.variants()]
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    st = torch.cuda.current_stream().cuda_stream
    rng = np.random.Generator(np.random.PCG64(7))
    stream = [SHAPES[i] for i in rng.integers(0, len(SHAPES), 70)]
    # every shape first appears in a fixed order of increasing size, so the fit has >= 3 keys early
    stream = SHAPES[:4] * 5 + stream
    probs, refs = {}, {}
    for s in SHAPES:
        m, n, k = s
        probs[s] = (device_matrix(gen.TAG_A, m, k), device_matrix(gen.TAG_B, k, n), torch.empty((m, n), device="cuda"))
        rows = np.arange(m) if m * n * k <= 1024 ** 3 else np.unique(np.linspace(0, m - 1, 12).astype(np.int64))
        Ar = gen.matrix_rows(gen.TAG_A, rows, k)
        B = gen.matrix(gen.TAG_B, k, n)
        refs[s] = (rows, Ar, B, og.gemm(Ar, B, alpha=1.5, beta=0.0))
    tmp = tempfile.mkdtemp()
    path = os.path.join(tmp, "perf.txt")
    modes = []
    try:
        for i, s in enumerate(stream):
            m, n, k = s
            A, B, C = probs[s]
            C.fill_(float("nan"))                       # beta = 0: C_in unread
            d = cm.make_desc(m, n, k, A=A, B=B, C_in=C, C_out=C, alpha=1.5, beta=0.0, compute=cm.COMPUTE_TF32,
                             stream=st)
            ctx.perf_save(path)
            orc = so.SelectorOracle(len(names), blocked=True, prune_pct=150)
            orc.hist = load_dump(path, names)
            elig = ctx.eligible(d)
            key = (m, n, k, so.F32, so.COMPUTE_TF32, 0, 1)
            lb = [so.SelectorOracle.static_lb_ns(lb_class(names[v]), key, sms) for v in elig]
            (ev, emode), _ = expected(orc, key, elig, lb)
            r = ctx.run(d)
            assert r.status == 0
            assert (r.variant, r.mode) == (ev, emode), (i, s, names[r.variant], r.mode, names[ev], emode)
            modes.append(r.mode)
            rows, Ar, Bh, ref = refs[s]
            got = C[torch.as_tensor(rows, device="cuda")].double().cpu().numpy()
            tf32 = names[r.variant].startswith("tc_tf32")
            assert_parity(got, ref, Ar, Bh, None, 1.5, 0.0, "f32", tf32, 5e-3 if tf32 else 1e-5,
                          (i, s, names[r.variant]), tc=names[r.variant].startswith("tc_"))
    finally:
        ctx.terminate()
    # the generalisation did its job: shapes first seen after the fit decided without calibrating
    # every variant (PREDICT decisions exist), and the stream settles into model / predict mode.
    # (R37 exploration — one warm-up + one timed run of a variant predicted within 1.5x of the
    # measured best — may still fall on any single late task, so the tail is judged as a whole.)
    assert cm.MODE_PREDICT in modes
    tail = modes[-30:]
    settled = sum(md in (cm.MODE_MODEL, cm.MODE_PREDICT) for md in tail)
    assert settled >= 0.7 * len(tail), modes
