"""The FP32-accuracy tensor-core form `tc_f32x3` (precision class F32_SPLIT, R38) on the
GPU (-m gpu), against the FP64 oracle through the C ABI.

The paper's arrays are FP32 (PAPER.md P:78 [§2.1], P:201-205 [Table 2, SGEMM variants]); this
variant reaches FP32 accuracy on TF32 tensor cores by splitting every operand into TF32 hi + lo
and summing hi*hi + hi*lo + lo*hi.  It is held to the strict-FP32 bounds — rel-Fro <= 1e-5 with
no tensor-core widening, and every element inside the componentwise FP32 dot-product bound —
on shapes that cross its 1024-k accumulation chunks, ragged tiles, transB, beta = 0 with NaN
C_in, and the 8192^3 bench target (sampled rows); integer inputs are bitwise exact.  On the same
data the plain TF32 variant misses 1e-5 by orders of magnitude (so the split is what does it).
"""
import numpy as np
import pytest

import gen
from oracle import gemm as og

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from tests._gpu_util import assert_parity, device_matrix, to_device, to_host_f64  # noqa: E402

cm = pytest.importorskip("paper_2311_03543_b200.compar")


@pytest.fixture(scope="module")
def ctx():
    c = cm.Compar()
    yield c
    c.terminate()


def vid(ctx, name):
    return [n for n, _ in ctx.variants()].index(name)


def run(ctx, name, m, n, k, compute, dist=gen.DIST_U, beta=0.5, transB=0, seed=21):
    A = gen.matrix(gen.TAG_A, m, k, dist, "f32", seed=seed)
    B = gen.matrix(gen.TAG_B, k, n, dist, "f32", seed=seed)
    C0 = gen.matrix(gen.TAG_C, m, n, dist, "f32", seed=seed)
    lda = k + (-k) % 4
    ldb = (k if transB else n) + (-(k if transB else n)) % 4
    Ad = to_device(A, "f32", lda)
    Bd = to_device(np.ascontiguousarray(B.T) if transB else B, "f32", ldb)
    Cd = to_device(C0, "f32", n + (-n) % 4)
    if beta == 0.0:
        Cd.fill_(float("nan"))
    alpha = 2.0 if dist == gen.DIST_I else 1.5
    d = cm.make_desc(m, n, k, A=Ad, B=Bd, C_in=Cd, C_out=Cd, lda=lda, ldb=ldb, ldc_in=Cd.shape[1],
                     ldc_out=Cd.shape[1], alpha=alpha, beta=beta, compute=compute, transB=transB,
                     stream=torch.cuda.current_stream().cuda_stream, variant_hint=vid(ctx, name))
    r = ctx.run(d)
    assert r.status == 0 and r.variant == vid(ctx, name)
    got = to_host_f64(Cd[:, :n])
    return got, og.gemm(A, B, C0, alpha=alpha, beta=beta), (A, B, C0, alpha, beta)


SHAPES = [(64, 64, 64), (300, 520, 1000), (129, 257, 1024), (129, 257, 1025), (257, 300, 2100),
          (1000, 777, 333), (1, 300, 4097), (513, 1, 3000), (2048, 2048, 2048)]


@pytest.mark.parametrize("transB", [0, 1])
@pytest.mark.parametrize("beta", [0.5, 0.0])
@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s)))
def test_f32x3_strict_fp32_bounds(ctx, shape, beta, transB):
    m, n, k = shape
    got, ref, (A, B, C0, alpha, beta_) = run(ctx, "tc_f32x3", m, n, k, cm.COMPUTE_F32_SPLIT, beta=beta, transB=transB)
    assert np.isfinite(got).all()
    assert_parity(got, ref, A, B, C0, alpha, beta_, "f32", False, 1e-5, ("tc_f32x3", shape), tc=False)


@pytest.mark.parametrize("shape", [(200, 300, 517), (129, 257, 2500), (1000, 384, 4100)],
                         ids=lambda s: "x".join(map(str, s)))
def test_f32x3_exact_integers(ctx, shape):
    """Integers in {-2..2} are TF32 values: lo = 0, every partial sum an exact integer — bitwise,
    across 1..5 accumulation chunks."""
    m, n, k = shape
    got, ref, _ = run(ctx, "tc_f32x3", m, n, k, cm.COMPUTE_F32_SPLIT, dist=gen.DIST_I, beta=-1.0)
    np.testing.assert_array_equal(got, ref)


def test_f32x3_beats_tf32_accuracy(ctx):
    """Same inputs: tc_tf32 (one TF32 product) sits far above 1e-5; tc_f32x3 inside it, >= 30x closer."""
    m, n, k = 512, 512, 2048
    g1, ref, args = run(ctx, "tc_f32x3", m, n, k, cm.COMPUTE_F32_SPLIT)
    g2, _, _ = run(ctx, "tc_tf32_2sm", m, n, k, cm.COMPUTE_TF32)
    e1, e2 = og.rel_fro(g1, ref), og.rel_fro(g2, ref)
    assert e1 <= 1e-5 < e2 and e2 >= 30 * e1, (e1, e2)


def test_f32x3_full_size_sampled(ctx):
    """The bench target (config 3 under F32_SPLIT, 8192^3): sampled full rows against the oracle."""
    m = n = k = 8192
    A = device_matrix(gen.TAG_A, m, k)
    B = device_matrix(gen.TAG_B, k, n)
    C = device_matrix(gen.TAG_C, m, n)
    d = cm.make_desc(m, n, k, A=A, B=B, C_in=C, C_out=C, alpha=1.5, beta=0.5, compute=cm.COMPUTE_F32_SPLIT,
                     variant_hint=vid(ctx, "tc_f32x3"), stream=torch.cuda.current_stream().cuda_stream)
    assert ctx.run(d).status == 0
    rows = np.unique(np.concatenate([[0, 127, 128, 255, 256, m // 2, m - 1],
                                     np.random.default_rng(4).integers(0, m, 9)])).astype(np.int64)
    Ar = gen.matrix_rows(gen.TAG_A, rows, k)
    Bf = gen.matrix(gen.TAG_B, k, n)
    C0 = gen.matrix_rows(gen.TAG_C, rows, n)
    ref = og.gemm(Ar, Bf, C0, alpha=1.5, beta=0.5)
    got = C[torch.as_tensor(rows, device="cuda")].double().cpu().numpy()
    assert_parity(got, ref, Ar, Bf, C0, 1.5, 0.5, "f32", False, 1e-5, "tc_f32x3 8192^3", tc=False)


def test_f32x3_eligibility(ctx):
    """Eligible only under F32_SPLIT, from K >= 64, TMA-aligned, device memory; F32_SPLIT also
    admits the FFMA variants (so every F32_SPLIT descriptor has a variant), never plain TF32 ones."""
    names = [n for n, _ in ctx.variants()]
    A = torch.zeros((256, 256), device="cuda")
    B = torch.zeros((256, 256), device="cuda")
    C = torch.zeros((256, 256), device="cuda")
    el = lambda d: sorted(names[v] for v in ctx.eligible(d))  # noqa: E731
    d = cm.make_desc(256, 256, 256, A=A, B=B, C_in=C, C_out=C, compute=cm.COMPUTE_F32_SPLIT)
    assert el(d) == sorted(["simt_f32", "tma_f32", "tc_f32x3"])
    d63 = cm.make_desc(256, 256, 63, A=A, B=B, C_in=C, C_out=C, lda=256, ldb=256, compute=cm.COMPUTE_F32_SPLIT)
    assert "tc_f32x3" not in el(d63)
    for cp in (cm.COMPUTE_F32_STRICT, cm.COMPUTE_TF32):
        assert "tc_f32x3" not in el(cm.make_desc(256, 256, 256, A=A, B=B, C_in=C, C_out=C, compute=cp))
    Ah, Bh, Ch = (torch.zeros((256, 256)).pin_memory() for _ in range(3))
    dh = cm.make_desc(256, 256, 256, A=Ah, B=Bh, C_in=Ch, C_out=Ch, compute=cm.COMPUTE_F32_SPLIT, mem=cm.MEM_HOST)
    assert "tc_f32x3" not in el(dh)


def test_f32x3_panels_bitwise(ctx):
    """Local row panels P in {2, 3}: each panel re-splits its operands; chunks depend on K only,
    so C is bitwise the P = 1 result."""
    m, n, k = 1000, 384, 2100
    A = device_matrix(gen.TAG_A, m, k)
    B = device_matrix(gen.TAG_B, k, n)
    C0 = device_matrix(gen.TAG_C, m, n)
    outs = []
    for P in (1, 2, 3):
        Cd = C0.clone()
        d = cm.make_desc(m, n, k, A=A, B=B, C_in=Cd, C_out=Cd, alpha=1.5, beta=0.5, compute=cm.COMPUTE_F32_SPLIT,
                         panels=P, variant_hint=vid(ctx, "tc_f32x3"), stream=torch.cuda.current_stream().cuda_stream)
        assert ctx.run(d).status == 0
        outs.append(Cd.cpu())
    for o in outs[1:]:
        assert torch.equal(o, outs[0])


def test_f32x3_workspace_released_at_last_terminate(tmp_path):
    """The per-stream operand workspace (12 (mk + kn) bytes: 3.2 GB at 8192^3) is freed when the
    last context terminates (a separate process, so no other test's context is alive)."""
    import subprocess
    import sys
    script = tmp_path / "ws.py"
    script.write_text(
        "import sys, torch\n"
        f"sys.path.insert(0, {str(__import__('os').path.dirname(__import__('os').path.dirname(__file__)))!r})\n"
        "import gen\n"
        "from gen.device import device_matrix\n"
        "from paper_2311_03543_b200 import compar as cm\n"
        "m = n = k = 8192\n"
        "A, B, C = device_matrix(gen.TAG_A, m, k), device_matrix(gen.TAG_B, k, n), device_matrix(gen.TAG_C, m, n)\n"
        "ctx = cm.Compar()\n"
        "names = [v for v, _ in ctx.variants()]\n"
        "d = cm.make_desc(m, n, k, A=A, B=B, C_in=C, C_out=C, alpha=1.0, beta=0.5, compute=cm.COMPUTE_F32_SPLIT,\n"
        "                 variant_hint=names.index('tc_f32x3'), stream=torch.cuda.current_stream().cuda_stream)\n"
        "assert ctx.run(d).status == 0\n"
        "torch.cuda.synchronize()\n"
        "f0 = torch.cuda.mem_get_info()[0]\n"
        "ctx.terminate()\n"
        "f1 = torch.cuda.mem_get_info()[0]\n"
        "print(f1 - f0)\n")
    out = subprocess.run([sys.executable, str(script)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    freed = int(out.stdout.strip().splitlines()[-1])
    assert freed >= 12 * (8192 * 8192 * 2) * 0.95, freed
