"""World-mode (multi-GPU) path on one GPU (-m gpu): the N-slab broadcast pipeline is exercised in
loopback (COMPAR_BCAST_LOOPBACK=1: the NCCL broadcast of each slab is emulated by a D2D copy on
the comm stream, the GEMM consumes the received slabs exactly as a non-root rank does).  The
result must be BITWISE equal to the plain single-launch call (every C element still sums its
full K in order — DESIGN.md §6), for row-major and transposed B and ragged slab widths."""
import os

import numpy as np
import pytest

import gen

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from gen.device import device_matrix  # noqa: E402
from oracle import gemm as og  # noqa: E402
from tests._gpu_util import assert_parity  # noqa: E402

cm = pytest.importorskip("paper_2311_03543_b200.compar")


@pytest.fixture(scope="module")
def loop_ctx():
    old = os.environ.get("COMPAR_BCAST_LOOPBACK")
    os.environ["COMPAR_BCAST_LOOPBACK"] = "1"
    ctxs = {}

    def get(chunks):
        if chunks not in ctxs:
            ctxs[chunks] = cm.Compar(bcast_chunks=chunks)
        return ctxs[chunks]
    yield get
    for c in ctxs.values():
        c.terminate()
    if old is None:
        os.environ.pop("COMPAR_BCAST_LOOPBACK", None)
    else:
        os.environ["COMPAR_BCAST_LOOPBACK"] = old


CASES = [("tc_bf16", 1000, 1000, 704, 0), ("tc_bf16", 1000, 1000, 704, 1), ("tc_bf16_2sm", 777, 2048, 512, 0),
         ("tc_tf32", 300, 1280, 256, 0), ("tc_tf32_2sm", 512, 1030, 300, 1), ("simt_f32", 200, 600, 100, 0),
         # the wide pair kernel: N a multiple of 512 -> one fused launch waiting per slab on device flags
         ("tc_bf16_2sm_w", 1000, 2048, 704, 0), ("tc_bf16_2sm_w", 777, 3072, 304, 1),
         ("tc_tf32_2sm_w", 600, 1536, 260, 0), ("tc_tf32_2sm_w", 520, 1024, 512, 1),
         ("tc_bf16_2sm_w", 640, 1000, 512, 0),          # (N not a multiple of 512: per-slab launches)
         # FP32 accuracy (R38): one launch per slab, each re-splitting the panel's A and the slab
         ("tc_f32x3", 600, 1280, 1100, 0), ("tc_f32x3", 520, 1536, 2100, 1)]


@pytest.mark.parametrize("chunks", [1, 3, 4])
@pytest.mark.parametrize("name,m,n,k,tb", CASES)
def test_loopback_slab_pipeline_bitwise(loop_ctx, chunks, name, m, n, k, tb):
    ctx = loop_ctx(chunks)
    names = [v for v, _ in ctx.variants()]
    bf = "bf16" in name
    dt = "bf16" if bf else "f32"
    compute = cm.COMPUTE_BF16 if bf else (cm.COMPUTE_TF32 if "tf32" in name else
                                          cm.COMPUTE_F32_SPLIT if name == "tc_f32x3" else cm.COMPUTE_F32_STRICT)
    A = device_matrix(gen.TAG_A, m, k, dtype=dt)
    B = device_matrix(gen.TAG_B, k, n, dtype=dt, transposed=bool(tb))
    C0 = device_matrix(gen.TAG_C, m, n)
    outs = []
    for world in (0, 1):
        Cd = C0.clone()
        d = cm.make_desc(m, n, k, A=A, B=B, C_in=Cd, C_out=Cd, ldb=(k if tb else n), alpha=1.5, beta=0.5,
                         in_dtype=cm.BF16 if bf else cm.F32, compute=compute, transB=tb, world=world,
                         variant_hint=names.index(name))
        r = ctx.run(d)
        assert r.status == 0
        if world:
            assert r.total_ns >= r.ns
        outs.append(Cd.cpu())
    assert torch.equal(outs[0], outs[1])
    if chunks == 4:   # and the pipeline result matches the oracle
        got = outs[1].double().numpy()
        Ah, Bh, Ch = gen.matrix(gen.TAG_A, m, k, dtype=dt), gen.matrix(gen.TAG_B, k, n, dtype=dt), gen.matrix(gen.TAG_C, m, n)
        ref = og.gemm(Ah, Bh, Ch, alpha=1.5, beta=0.5, dtype=dt)
        tf32 = name.startswith("tc_tf32")
        assert_parity(got, ref, Ah, Bh, Ch, 1.5, 0.5, dt, tf32, 5e-3 if tf32 else 1e-5, name,
                      tc=name.startswith("tc_") and name != "tc_f32x3")


@pytest.mark.parametrize("name,m,n,k,tb", [("tc_bf16_2sm_w", 4096, 4096, 1024, 0), ("tc_tf32_2sm_w", 3072, 4096, 520, 1),
                                            ("tc_bf16_2sm_w", 4096, 8192, 2048, 0)])
def test_loopback_fused_with_helper_launch_bitwise(name, m, n, k, tb):
    """COMPAR_BCAST_LOOPBACK=2: the loopback pipeline also leaves bcast_reserve_sms SMs free while
    the 'broadcast' runs, so the wide kernel's main launch runs on fewer SMs and a helper launch on
    the library's aux stream joins after the broadcast, sharing the tile counter; plus several
    tasks back to back (counter re-arm across the cooperating launches).  C bitwise = plain call."""
    old = os.environ.get("COMPAR_BCAST_LOOPBACK")
    os.environ["COMPAR_BCAST_LOOPBACK"] = "2"
    try:
        ctx = cm.Compar(bcast_chunks=4, bcast_ctas=8)
    finally:
        if old is None:
            os.environ.pop("COMPAR_BCAST_LOOPBACK", None)
        else:
            os.environ["COMPAR_BCAST_LOOPBACK"] = old
    try:
        names = [v for v, _ in ctx.variants()]
        bf = "bf16" in name
        dt = "bf16" if bf else "f32"
        A = device_matrix(gen.TAG_A, m, k, dtype=dt)
        B = device_matrix(gen.TAG_B, k, n, dtype=dt, transposed=bool(tb))
        C0 = device_matrix(gen.TAG_C, m, n)
        kw = dict(ldb=(k if tb else n), alpha=1.5, beta=0.5, in_dtype=cm.BF16 if bf else cm.F32,
                  compute=cm.COMPUTE_BF16 if bf else cm.COMPUTE_TF32, transB=tb, variant_hint=names.index(name))
        Cp = C0.clone()
        ctx.run(cm.make_desc(m, n, k, A=A, B=B, C_in=Cp, C_out=Cp, **kw))
        s0 = ctx.stats()
        outs = []
        for _ in range(3):
            Cw = C0.clone()
            r = ctx.run(cm.make_desc(m, n, k, A=A, B=B, C_in=Cw, C_out=Cw, world=1, **kw))
            assert r.status == 0 and r.bcast_ns > 0
            outs.append(Cw)
        assert ctx.stats().launches - s0.launches == 6          # main + helper per task
        for o in outs:
            assert torch.equal(o, Cp)
    finally:
        ctx.terminate()


@pytest.mark.parametrize("tb", [0, 1])
def test_loopback_through_nccl_one_rank(tb):
    """Same pipeline, but every slab goes through ncclBroadcast on a real 1-rank communicator
    (send = packed slab, recv = replica slab) and every harvested sample through ncclAllReduce —
    the NCCL call sites of the N-GPU path, exercised on one GPU, with the selector calibrating."""
    old = os.environ.get("COMPAR_BCAST_LOOPBACK")
    os.environ["COMPAR_BCAST_LOOPBACK"] = "1"
    try:
        ctx = cm.Compar(bcast_chunks=4)
        ctx.comm_init(1, 0, cm.comm_unique_id())
    finally:
        if old is None:
            os.environ.pop("COMPAR_BCAST_LOOPBACK", None)
        else:
            os.environ["COMPAR_BCAST_LOOPBACK"] = old
    try:
        m, n, k = 1024, 2048, 512
        A = device_matrix(gen.TAG_A, m, k, dtype="bf16")
        B = device_matrix(gen.TAG_B, k, n, dtype="bf16", transposed=bool(tb))
        C0 = device_matrix(gen.TAG_C, m, n)
        kw = dict(ldb=(k if tb else n), alpha=1.5, beta=0.5, in_dtype=cm.BF16, compute=cm.COMPUTE_BF16, transB=tb)
        n_bf16 = len(ctx.eligible(cm.make_desc(m, n, k, A=A, B=B, C_in=C0, C_out=C0, world=1, **kw)))
        for _ in range(4 * n_bf16 + 2):   # calibration (1 warm-up + 3 per variant), then model mode, via world=1
            Cw = C0.clone()
            r = ctx.run(cm.make_desc(m, n, k, A=A, B=B, C_in=Cw, C_out=Cw, world=1, **kw))
            assert r.status == 0 and r.bcast_ns >= 0
        assert r.mode == cm.MODE_MODEL
        Cp = C0.clone()
        ctx.run(cm.make_desc(m, n, k, A=A, B=B, C_in=Cp, C_out=Cp, variant_hint=r.variant, **kw))
        assert torch.equal(Cw, Cp)
    finally:
        ctx.terminate()


def test_loopback_world_host_memory(loop_ctx):
    """World mode + HOST buffers (the e2e path of bench.py at N > 1) through the slab pipeline."""
    ctx = loop_ctx(4)
    m, n, k = 640, 1536, 512
    A = gen.matrix(gen.TAG_A, m, k, dtype="bf16")
    B = gen.matrix(gen.TAG_B, k, n, dtype="bf16")
    C0 = gen.matrix(gen.TAG_C, m, n)
    Ah = torch.from_numpy(A.view(np.int16)).view(torch.bfloat16).pin_memory()
    Bh = torch.from_numpy(B.view(np.int16)).view(torch.bfloat16).pin_memory()
    Ch = torch.from_numpy(C0.copy()).pin_memory()
    d = cm.make_desc(m, n, k, A=Ah, B=Bh, C_in=Ch, C_out=Ch, alpha=1.5, beta=0.5, in_dtype=cm.BF16,
                     compute=cm.COMPUTE_BF16, mem=cm.MEM_HOST, world=1)
    ctx.run(d)
    ref = og.gemm(A, B, C0, alpha=1.5, beta=0.5, dtype="bf16")
    assert_parity(Ch.double().numpy(), ref, A, B, C0, 1.5, 0.5, "bf16", False, 1e-5, "world host", tc=True)
