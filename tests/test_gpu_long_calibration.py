"""R39 on the GPU (-m gpu): a key whose variants' static lower bounds are >= 10 ms (32768 x 32768 x
16384 BF16: 15.6 ms at the datasheet peak) calibrates each tensor-core variant with 6 warm-up runs
before its 3 timed ones, so the timed samples see the power-capped steady state; every decision
(variant, mode) equals oracle/selector.py's, fed with the runtime's own history (compar_perf_save)
before each submit, and the calibration ends in model mode on the smallest mean."""
import os
import tempfile

import pytest

import gen
from oracle import selector as so

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from gen.device import fill  # noqa: E402

cm = pytest.importorskip("paper_2311_03543_b200.compar")


def load_dump(path, names):
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
    if name.startswith("tc_bf16"):
        return "bf16"
    return "ffma" if name == "simt_bf16" else None


def test_long_kernel_calibration_matches_oracle():
    m, n, k = 32768, 32768, 16384
    st = torch.cuda.current_stream().cuda_stream
    A = torch.empty((m, k), dtype=torch.bfloat16, device="cuda")
    B = torch.empty((k, n), dtype=torch.bfloat16, device="cuda")
    C = torch.empty((m, n), device="cuda")
    fill(A.data_ptr(), "bf16", m, k, k, gen.TAG_A, stream=st)
    fill(B.data_ptr(), "bf16", k, n, n, gen.TAG_B, stream=st)
    fill(C.data_ptr(), "f32", m, n, n, gen.TAG_C, stream=st)
    torch.cuda.synchronize()
    ctx = cm.Compar()
    names = [nm for nm, _ in ctx.variants()]
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    path = os.path.join(tempfile.mkdtemp(), "perf.txt")
    d = cm.make_desc(m, n, k, A=A, B=B, C_in=C, C_out=C, alpha=1.0, beta=0.5, in_dtype=cm.BF16,
                     compute=cm.COMPUTE_BF16, stream=st)
    key = (m, n, k, so.BF16, so.COMPUTE_BF16, 0, 0)
    trace = []
    try:
        elig = ctx.eligible(d)
        lb = [so.SelectorOracle.static_lb_ns(lb_class(names[v]), key, sms) for v in elig]
        for _ in range(40):
            ctx.perf_save(path)
            orc = so.SelectorOracle(len(names), blocked=True)
            orc.hist = load_dump(path, names)
            ev, emode = orc.decide(key, elig, lb)
            r = ctx.run(d)
            assert r.status == 0
            assert (r.variant, r.mode) == (ev, emode), (len(trace), names[r.variant], r.mode, names[ev], emode)
            trace.append((names[r.variant], r.mode))
            if r.mode == cm.MODE_MODEL:
                break
    finally:
        ctx.terminate()
    assert trace[-1][1] == cm.MODE_MODEL
    for name in ("tc_bf16", "tc_bf16_2sm", "tc_bf16_2sm_w"):
        modes = [md for nm, md in trace if nm == name and md in (cm.MODE_WARMUP, cm.MODE_CALIB)]
        assert modes == [cm.MODE_WARMUP] * 6 + [cm.MODE_CALIB] * 3, (name, modes)
    assert not any(nm == "simt_bf16" for nm, _ in trace)          # pruned by its lower bound (R32)
