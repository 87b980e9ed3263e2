"""GPU parity of every built-in variant against the FP64 oracle, through the C ABI (-m gpu).

Tolerances (BASELINE.json north_star; R8): max relative Frobenius error 1e-5 for
the strict-FP32 variants (simt_f32, tma_f32) and for every BF16 variant (the oracle consumes the
same RNE-quantised BF16 values, so the only error left is FP32 accumulation: SURVEY c7) — for the
BF16 tensor-core variants max(1e-5, K * 2^-27), because the tcgen05 accumulator truncates
(tests/_gpu_util.tc_accum_tol, R33) — and 5e-3 only where TF32 truncation applies
(tc_tf32*).  Every non-integer comparison ALSO checks each element
against the componentwise FP32-accumulation bound (oracle.gemm.elementwise_bound, TF32 operand
term for tc_tf32*).  Integer-valued inputs (distribution I) must match BITWISE for every variant
(every partial sum is an exact integer < 2^24, SURVEY §8(c) "Exact integers").
"""
import math

import numpy as np
import pytest

import gen
from oracle import gemm as og

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from tests._gpu_util import assert_parity, device_matrix, to_device, to_host_f64  # noqa: E402

cm = pytest.importorskip("paper_2311_03543_b200.compar")

VARIANTS = {"simt_f32": (cm.F32, cm.COMPUTE_F32_STRICT, 1e-5),
            "tma_f32": (cm.F32, cm.COMPUTE_F32_STRICT, 1e-5),
            "tc_tf32": (cm.F32, cm.COMPUTE_TF32, 5e-3),
            "tc_bf16": (cm.BF16, cm.COMPUTE_BF16, 1e-5),
            "tc_tf32_2sm": (cm.F32, cm.COMPUTE_TF32, 5e-3),
            "tc_bf16_2sm": (cm.BF16, cm.COMPUTE_BF16, 1e-5),
            "tc_tf32_2sm_w": (cm.F32, cm.COMPUTE_TF32, 5e-3),
            "tc_bf16_2sm_w": (cm.BF16, cm.COMPUTE_BF16, 1e-5),
            "tc_tf32_sk": (cm.F32, cm.COMPUTE_TF32, 5e-3),
            "tc_bf16_sk": (cm.BF16, cm.COMPUTE_BF16, 1e-5),
            "tc_tf32_ck": (cm.F32, cm.COMPUTE_TF32, 5e-3),
            "tc_bf16_ck": (cm.BF16, cm.COMPUTE_BF16, 1e-5),
            # FP32 accumulation of exactly-widened BF16 operands: held to the strict-FP32 bound
            "simt_bf16": (cm.BF16, cm.COMPUTE_BF16, 1e-5),
            # FP32 accuracy from three TF32 products per product (R38): the strict-FP32 bounds
            "tc_f32x3": (cm.F32, cm.COMPUTE_F32_SPLIT, 1e-5)}

SHAPES = [(1, 1, 1), (7, 13, 5), (64, 64, 64), (65, 127, 129), (129, 257, 70), (128, 256, 64),
          (300, 520, 1000), (1000, 777, 333), (257, 1, 100), (1, 300, 4097)]


def sk_splits(m, n, k, bf16):
    """Mirror of tc_splitk_splits (kernels.h): K splits of the tc_*_sk variant, 0 = not eligible."""
    kb = -(-k // (64 if bf16 else 32))
    s = min(8, kb // 32)
    tiles = -(-m // 256) * -(-n // 256)
    return s if s >= 2 and tiles * s * 256 * 256 * 4 <= (1 << 30) else 0


def ineligible_reason(name, m, n, k):
    """The eligibility rules of the K-split variants and tc_f32x3 (kernels.h, R38),
    restated: a case they exclude is checked as a refusal instead of a product."""
    if name.endswith("_sk") and not sk_splits(m, n, k, "bf16" in name):
        return f"{name} needs >= 64 k-blocks (K = {k})"
    if name.endswith("_ck") and k <= (64 if "bf16" in name else 32):
        return f"{name} needs >= 2 k-blocks (K = {k})"
    if name == "tc_f32x3" and k < 64:
        return "tc_f32x3 needs K >= 64 (DESIGN.md R38)"
    return None


def assert_refused(ctx, d, name):
    """An ineligible variant is outside E (§8(c) step 1) and a task hinted to it is refused
    (E_INVALID "not eligible") before anything launches: never run on a shape it does not support."""
    v = vid(ctx, name)
    assert v not in ctx.eligible(d)
    d.variant_hint = v
    with pytest.raises(cm.ComparError) as ei:
        ctx.run(d)
    assert ei.value.status == cm.E_INVALID and "not eligible" in str(ei.value), ei.value
    return Refused(name)


class Refused:
    """run_case's result for a refused (ineligible) case: no C was produced, so there is nothing
    to compare — the refusal itself was the check."""

    def __init__(self, name):
        self.name = name
        self.got = self.ref = np.zeros((0,))

    def check(self):
        return None


@pytest.fixture(scope="module")
def ctx():
    c = cm.Compar()
    yield c
    c.terminate()


def vid(ctx, name):
    return [n for n, _ in ctx.variants()].index(name)


def run_case(ctx, name, m, n, k, dist=gen.DIST_U, beta=0.5, transB=0, pad=8, seed=11, ldc_pad=4):
    refused = ineligible_reason(name, m, n, k)
    dtype_id, compute, tol = VARIANTS[name]
    dt = "bf16" if dtype_id == cm.BF16 else "f32"
    A = gen.matrix(gen.TAG_A, m, k, dist, dt, seed=seed)
    B = gen.matrix(gen.TAG_B, k, n, dist, dt, seed=seed)
    C0 = gen.matrix(gen.TAG_C, m, n, dist, "f32", seed=seed)
    lda = k + (-k) % pad
    ldb_cols = k if transB else n
    ldb = ldb_cols + (-ldb_cols) % pad
    ldc = n + (-n) % 4 if ldc_pad == 4 else n + ldc_pad
    Ad = to_device(A, dt, lda)
    Bd = to_device(np.ascontiguousarray(B.T) if transB else B, dt, ldb)
    Cd = to_device(C0, "f32", ldc)
    if beta == 0.0:
        Cd.fill_(float("nan"))
    alpha = 1.5 if dist != gen.DIST_I else 2.0
    d = cm.make_desc(m, n, k, A=Ad, B=Bd, C_in=Cd, C_out=Cd, lda=lda, ldb=ldb, ldc_in=ldc, ldc_out=ldc,
                     alpha=alpha, beta=beta, in_dtype=dtype_id, compute=compute, transB=transB,
                     stream=torch.cuda.current_stream().cuda_stream, variant_hint=vid(ctx, name))
    if refused:
        return assert_refused(ctx, d, name)
    rep = ctx.run(d)
    assert rep.status == 0 and rep.variant == vid(ctx, name)
    got = to_host_f64(Cd[:, :n])
    ref = og.gemm(A, B, C0, alpha=alpha, beta=beta, dtype=dt)
    return Case(got, ref, tol, A, B, C0, alpha, beta, dt, is_tf32(name), name)


def is_tf32(name):
    return name.startswith("tc_tf32")


class Case:
    """One run: GPU result, oracle result, and what the parity checks need."""

    def __init__(self, got, ref, tol, A, B, C0, alpha, beta, dt, tf32, name):
        self.got, self.ref, self.tol = got, ref, tol
        self._args = (A, B, C0, alpha, beta, dt, tf32)
        self.name = name

    def check(self):
        A, B, C0, alpha, beta, dt, tf32 = self._args
        # (tc_f32x3 claims FP32 accuracy: no widening of the norm tolerance for tensor-core accumulation)
        return assert_parity(self.got, self.ref, A, B, C0, alpha, beta, dt, tf32, self.tol, self.name,
                             tc=self.name.startswith("tc_") and self.name != "tc_f32x3")


@pytest.mark.parametrize("name", list(VARIANTS))
@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s)))
def test_parity_uniform(ctx, name, shape):
    m, n, k = shape
    run_case(ctx, name, m, n, k).check()


@pytest.mark.parametrize("name", list(VARIANTS))
@pytest.mark.parametrize("transB", [0, 1])
@pytest.mark.parametrize("shape", [(64, 64, 64), (200, 300, 517), (129, 257, 1030)], ids=lambda s: "x".join(map(str, s)))
def test_parity_exact_integers(ctx, name, transB, shape):
    m, n, k = shape
    c = run_case(ctx, name, m, n, k, dist=gen.DIST_I, beta=-1.0, transB=transB)
    np.testing.assert_array_equal(c.got, c.ref)


@pytest.mark.parametrize("name", ["tc_tf32_2sm", "tc_bf16_2sm"])
@pytest.mark.parametrize("shape", [(300, 519, 1000), (777, 255, 129)], ids=lambda s: "x".join(map(str, s)))
@pytest.mark.parametrize("beta", [0.5, 0.0])
def test_2sm_row_store_epilogue(ctx, name, shape, beta):
    """tc_*_2sm with a C that TMA cannot move (ldc * 4 % 16 != 0): the launcher falls back to
    the per-thread row-store epilogue kernel (tc_gemm_2sm.cu); same tolerance."""
    m, n, k = shape
    run_case(ctx, name, m, n, k, beta=beta, ldc_pad=1).check()


@pytest.mark.parametrize("name", ["tc_tf32_2sm", "tc_bf16_2sm", "tc_tf32_2sm_w", "tc_bf16_2sm_w"])
@pytest.mark.parametrize("transB", [0, 1])
@pytest.mark.parametrize("beta", [0.5, 0.0])
def test_pair_kernels_ragged_tiles(ctx, name, transB, beta):
    """Several pair tiles plus ragged M/N/K tails through the TMA-epilogue pair kernels."""
    run_case(ctx, name, 777, 600, 333, beta=beta, transB=transB).check()


def check_rows(Cd, rows, k, n, beta, dt, name, tol):
    """Full rows `rows` of a device result against the oracle fed from the host generator."""
    got = Cd[torch.as_tensor(rows, device="cuda")].double().cpu().numpy()
    Ar, B = gen.matrix_rows(gen.TAG_A, rows, k, dtype=dt), gen.matrix(gen.TAG_B, k, n, dtype=dt)
    C0 = gen.matrix_rows(gen.TAG_C, rows, n)
    ref = og.gemm(Ar, B, C0, alpha=1.5, beta=beta, dtype=dt)
    assert_parity(got, ref, Ar, B, C0, 1.5, beta, dt, is_tf32(name), tol, name, tc=name.startswith("tc_"))


@pytest.mark.parametrize("name", ["tc_tf32_2sm_w", "tc_bf16_2sm_w"])
@pytest.mark.parametrize("shape,transB,beta", [((4096, 5120, 1000), 0, 0.5), ((4000, 5000, 200), 1, 0.0),
                                               ((8192, 8192, 2048), 0, 0.5)], ids=["multi-tile", "short-k-t", "8k"])
def test_wide_epilogue_overlap_bitwise(ctx, monkeypatch, name, shape, transB, beta):
    """The wide kernel's overlapped schedule (first D k-steps into accumulator half 0 only, then
    half 1, then both) sums every output element over k in the same order as D = 0, so C is BITWISE
    equal for every delay (incl. D >= the number of k-steps)."""
    dtype_id, compute, tol = VARIANTS[name]
    dt = "bf16" if dtype_id == cm.BF16 else "f32"
    m, n, k = shape
    A = device_matrix(gen.TAG_A, m, k, dtype=dt)
    B = device_matrix(gen.TAG_B, k, n, dtype=dt, transposed=bool(transB))
    C0 = device_matrix(gen.TAG_C, m, n)
    outs = []
    for delay in ("0", "12", "3", "1000"):
        monkeypatch.setenv("COMPAR_TCW_DELAY", delay)      # launcher knobs are read at compar_init
        with cm.Compar() as kctx:
            Cd = C0.clone()
            d = cm.make_desc(m, n, k, A=A, B=B, C_in=Cd, C_out=Cd, alpha=1.5, beta=beta, in_dtype=dtype_id,
                             compute=compute, transB=transB, ldb=k if transB else n, variant_hint=vid(kctx, name),
                             stream=torch.cuda.current_stream().cuda_stream)
            assert kctx.run(d).status == 0
        outs.append(Cd)
    for o in outs[1:]:
        assert torch.equal(outs[0], o)
    rows = np.unique(np.linspace(0, m - 1, 24).astype(np.int64))
    check_rows(outs[1], rows, k, n, beta, dt, name, tol)


@pytest.mark.parametrize("name", ["tc_tf32_sk", "tc_bf16_sk"])
@pytest.mark.parametrize("shape", [(300, 520, 5000), (777, 600, 8200), (256, 256, 65536), (1000, 64, 4160)],
                         ids=lambda s: "x".join(map(str, s)))
@pytest.mark.parametrize("transB,beta,dist", [(0, 0.5, gen.DIST_U), (1, 0.0, gen.DIST_U), (0, -1.0, gen.DIST_I)],
                         ids=["U", "U-t-b0", "I"])
def test_splitk_parity(ctx, name, shape, transB, beta, dist):
    """tc_*_sk: K cut into 2..8 ranges (K only), planes summed in split order by the reduce kernel;
    within tolerance on U(-1,1) and bitwise on integer inputs (all partial sums exact)."""
    m, n, k = shape
    c = run_case(ctx, name, m, n, k, dist=dist, beta=beta, transB=transB)
    if dist == gen.DIST_I:
        np.testing.assert_array_equal(c.got, c.ref)
    else:
        c.check()


@pytest.mark.parametrize("name", ["tc_tf32", "tc_bf16", "tma_f32", "tc_tf32_2sm", "tc_bf16_2sm"])
@pytest.mark.parametrize("transB", [0, 1])
def test_small_tile_instantiations_bitwise(ctx, monkeypatch, name, transB):
    """tc_* (1-SM) at tile widths 256 / 128 / 64 and tma_f32 at tiles 128 / 64 — the launcher
    picks one from the grid size — give BITWISE the same C (same k order per element), within
    tolerance of the oracle."""
    env, widths = {"tma_f32": ("COMPAR_TMA_TILE", ("128", "64")),
                   "tc_tf32_2sm": ("COMPAR_TC2_BN", ("256", "128")),
                   "tc_bf16_2sm": ("COMPAR_TC2_BN", ("256", "128"))}.get(name, ("COMPAR_TC1_BN", ("256", "128", "64")))
    outs = []
    for w in widths:
        monkeypatch.setenv(env, w)                          # launcher knobs are read at compar_init
        with cm.Compar() as kctx:
            c = run_case(kctx, name, 700, 900, 333, transB=transB)
        outs.append(c.got)
        c.check()
    for o in outs[1:]:
        np.testing.assert_array_equal(o, outs[0])


@pytest.mark.parametrize("name", list(VARIANTS))
def test_transB_and_beta0_nan(ctx, name):
    c = run_case(ctx, name, 190, 300, 260, transB=1, beta=0.0)
    assert np.isfinite(c.got).all()
    c.check()


@pytest.mark.parametrize("name", list(VARIANTS))
def test_positive_distribution(ctx, name):
    """P = U[0,1) exposes TF32 truncation bias (R6); still within 5e-3 (TF32) / 1e-5."""
    run_case(ctx, name, 256, 512, 2048, dist=gen.DIST_P).check()


def test_tma_variants_need_aligned_ld(ctx):
    """Eligibility filter: lda*4 % 16 != 0 removes tma_f32 and tc_tf32 from E."""
    m = n = k = 33
    A = torch.zeros((m, k), device="cuda")
    B = torch.zeros((k, n), device="cuda")
    Cm = torch.zeros((m, n), device="cuda")
    for name in ("tma_f32", "tc_tf32"):
        d = cm.make_desc(m, n, k, A=A, B=B, C_in=Cm, C_out=Cm, compute=cm.COMPUTE_TF32, variant_hint=vid(ctx, name))
        with pytest.raises(cm.ComparError):
            ctx.submit(d)
    d = cm.make_desc(m, n, k, A=A, B=B, C_in=Cm, C_out=Cm, compute=cm.COMPUTE_TF32)
    v, _ = ctx.select(d)
    assert v == vid(ctx, "simt_f32")


@pytest.mark.parametrize("name", list(VARIANTS))
def test_deterministic_rerun(ctx, name):
    a = run_case(ctx, name, 300, 400, 700, seed=5).got
    b = run_case(ctx, name, 300, 400, 700, seed=5).got
    np.testing.assert_array_equal(a, b)


def test_scale_paths(ctx):
    """k == 0 and alpha == 0: C = beta * C_in with A, B unread (BLAS rule R3)."""
    m, n = 70, 90
    C0 = gen.matrix(gen.TAG_C, m, n)
    for k, alpha in ((0, 1.5), (16, 0.0)):
        Cd = to_device(C0)
        A = torch.full((m, max(k, 1)), float("nan"), device="cuda")
        B = torch.full((max(k, 1), n), float("nan"), device="cuda")
        d = cm.make_desc(m, n, k, A=A, B=B, C_in=Cd, C_out=Cd, lda=max(k, 1), ldb=n, alpha=alpha, beta=-0.5)
        r = ctx.run(d)
        assert r.mode == cm.MODE_NOOP
        np.testing.assert_array_equal(to_host_f64(Cd), -0.5 * C0.astype(np.float64))


@pytest.mark.parametrize("name", list(VARIANTS))
def test_loopback_partition_bitwise_invariant(ctx, name):
    """Row panels P in {2, 3, 8} give C bitwise equal to P = 1 (a4 formula; the split-K variant's
    splits depend on K only)."""
    dtype_id, compute, _ = VARIANTS[name]
    dt = "bf16" if dtype_id == cm.BF16 else "f32"
    m, n, k = 1000, 384, 320 if not name.endswith("_sk") else 4160
    A = device_matrix(gen.TAG_A, m, k, dtype=dt)
    B = device_matrix(gen.TAG_B, k, n, dtype=dt)
    C0 = device_matrix(gen.TAG_C, m, n)
    outs = []
    for P in (1, 2, 3, 8):
        Cd = C0.clone()
        d = cm.make_desc(m, n, k, A=A, B=B, C_in=Cd, C_out=Cd, alpha=1.5, beta=0.5, in_dtype=dtype_id,
                         compute=compute, panels=P, variant_hint=vid(ctx, name),
                         stream=torch.cuda.current_stream().cuda_stream)
        r = ctx.run(d)
        assert r.npanels == sum(1 for a, b in zip(cm.partition_rows(m, P), cm.partition_rows(m, P)[1:]) if b > a)
        outs.append(Cd.cpu())
    for o in outs[1:]:
        assert torch.equal(o, outs[0])


def test_host_memory_mode_matches_device(ctx):
    """mem = HOST: the library stages pinned host buffers; result equals the device path bitwise."""
    m, n, k = 512, 768, 384
    A = gen.matrix(gen.TAG_A, m, k, dtype="bf16")
    B = gen.matrix(gen.TAG_B, k, n, dtype="bf16")
    C0 = gen.matrix(gen.TAG_C, m, n)
    Ah = torch.from_numpy(A.view(np.int16)).view(torch.bfloat16).pin_memory()
    Bh = torch.from_numpy(B.view(np.int16)).view(torch.bfloat16).pin_memory()
    Ch = torch.from_numpy(C0.copy()).pin_memory()
    d = cm.make_desc(m, n, k, A=Ah, B=Bh, C_in=Ch, C_out=Ch, alpha=1.5, beta=0.5, in_dtype=cm.BF16,
                     compute=cm.COMPUTE_BF16, mem=cm.MEM_HOST, variant_hint=vid(ctx, "tc_bf16"))
    r = ctx.run(d)
    assert r.status == 0 and r.total_ns >= r.ns > 0
    Cd = to_device(C0)
    d2 = cm.make_desc(m, n, k, A=to_device(A, "bf16"), B=to_device(B, "bf16"), C_in=Cd, C_out=Cd, alpha=1.5,
                      beta=0.5, in_dtype=cm.BF16, compute=cm.COMPUTE_BF16, variant_hint=vid(ctx, "tc_bf16"))
    ctx.run(d2)
    assert torch.equal(Ch, Cd.cpu())
    ref = og.gemm(A, B, C0, alpha=1.5, beta=0.5, dtype="bf16")
    assert_parity(Ch.double().numpy(), ref, A, B, C0, 1.5, 0.5, "bf16", False, 1e-5, "host-mode tc_bf16", tc=True)


@pytest.mark.parametrize("name", ["tc_bf16", "tc_tf32_2sm", "simt_f32"])
def test_host_pipeline_ragged_separate_cin(ctx, name):
    """mem = HOST with row chunks (copy/compute overlap), ragged m, C_in != C_out, padded ld."""
    dtype_id, compute, tol = VARIANTS[name]
    dt = "bf16" if dtype_id == cm.BF16 else "f32"
    m, n, k = 1000, 264, 136
    A = gen.matrix(gen.TAG_A, m, k, dtype=dt)
    B = gen.matrix(gen.TAG_B, k, n, dtype=dt)
    C0 = gen.matrix(gen.TAG_C, m, n)

    def host(x, ld):
        buf = np.zeros((x.shape[0], ld), dtype=x.dtype)
        buf[:, :x.shape[1]] = x
        t = torch.from_numpy(buf.view(np.int16)).view(torch.bfloat16) if x.dtype == np.uint16 else torch.from_numpy(buf)
        return t.pin_memory()
    Ah, Bh, Cih = host(A, k + 8), host(B, n + 8), host(C0, n + 4)
    Coh = torch.zeros((m, n + 12), dtype=torch.float32).pin_memory()
    d = cm.make_desc(m, n, k, A=Ah, B=Bh, C_in=Cih, C_out=Coh, lda=k + 8, ldb=n + 8, ldc_in=n + 4, ldc_out=n + 12,
                     alpha=1.5, beta=0.5, in_dtype=dtype_id, compute=compute, mem=cm.MEM_HOST,
                     variant_hint=vid(ctx, name))
    r = ctx.run(d)
    assert r.status == 0
    ref = og.gemm(A, B, C0, alpha=1.5, beta=0.5, dtype=dt)
    assert_parity(Coh[:, :n].double().numpy(), ref, A, B, C0, 1.5, 0.5, dt, is_tf32(name), tol, name,
                  tc=name.startswith("tc_"))
    assert torch.all(Coh[:, n:] == 0)


def test_world_size_one_nccl(ctx):
    """SPMD path with a 1-rank NCCL communicator: world = 1 equals the plain call."""
    c = cm.Compar()
    try:
        c.comm_init(1, 0, cm.comm_unique_id())
        m, n, k = 300, 512, 256
        A = device_matrix(gen.TAG_A, m, k, dtype="bf16")
        B = device_matrix(gen.TAG_B, k, n, dtype="bf16")
        C0 = device_matrix(gen.TAG_C, m, n)
        C1, C2 = C0.clone(), C0.clone()
        kw = dict(alpha=1.5, beta=0.5, in_dtype=cm.BF16, compute=cm.COMPUTE_BF16, variant_hint=vid(c, "tc_bf16"))
        c.run(cm.make_desc(m, n, k, A=A, B=B, C_in=C1, C_out=C1, world=1, **kw))
        c.run(cm.make_desc(m, n, k, A=A, B=B, C_in=C2, C_out=C2, **kw))
        assert torch.equal(C1, C2)
    finally:
        c.terminate()


@pytest.mark.parametrize("name,shape", [("tc_bf16", (8192, 8192, 8192)), ("tc_tf32", (8192, 8192, 8192)),
                                        ("tc_bf16_2sm", (8192, 8192, 8192)), ("tc_tf32_2sm", (8192, 8192, 8192)),
                                        ("tc_bf16_2sm", (32768, 32768, 32768)), ("tc_bf16_2sm", (65536, 256, 4096)),
                                        ("tc_bf16_2sm_w", (32768, 32768, 32768)), ("tc_tf32_2sm_w", (8192, 8192, 8192)),
                                        ("tc_bf16_2sm_w", (65536, 256, 4096)),
                                        ("tc_bf16", (65536, 256, 4096)), ("tc_tf32", (65536, 256, 4096)),
                                        ("tc_bf16", (32768, 32768, 32768)),
                                        ("tc_tf32_sk", (1024, 1024, 8192)), ("tc_bf16_sk", (2048, 2048, 32768))])
def test_full_size_sampled(ctx, name, shape):
    """BASELINE.json full sizes in the bench launch configuration; checked on a sampled
    sub-block (rows {0, 127, 128, m/2, m-1} + 27 random rows, columns {0, 255, 256, n-1} + 28
    random columns) against the oracle fed from the HOST generator (the device twin is pinned
    bitwise to it in tests/test_gpu_runtime.py::test_device_generator_matches_host_bitwise)."""
    dtype_id, compute, tol = VARIANTS[name]
    dt = "bf16" if dtype_id == cm.BF16 else "f32"
    m, n, k = shape
    A = device_matrix(gen.TAG_A, m, k, dtype=dt)
    B = device_matrix(gen.TAG_B, k, n, dtype=dt)
    Cd = device_matrix(gen.TAG_C, m, n)
    d = cm.make_desc(m, n, k, A=A, B=B, C_in=Cd, C_out=Cd, alpha=1.5, beta=0.5, in_dtype=dtype_id,
                     compute=compute, variant_hint=vid(ctx, name), stream=torch.cuda.current_stream().cuda_stream)
    ctx.run(d)
    rng = np.random.default_rng(1)
    rows = np.unique(np.concatenate([[0, m - 1, 127, 128, m // 2], rng.integers(0, m, 27)]))
    cols = np.unique(np.concatenate([[0, n - 1, 255, min(256, n - 1)], rng.integers(0, n, 28)]))
    got = Cd[torch.as_tensor(rows, device="cuda")][:, torch.as_tensor(cols, device="cuda")].double().cpu().numpy()
    Ar = gen.matrix_rows(gen.TAG_A, rows, k, dtype=dt)
    Bc = gen.matrix_cols(gen.TAG_B, k, cols, dtype=dt)
    C0 = gen.matrix_entries(gen.TAG_C, rows, cols)
    ref = og.gemm(Ar, Bc, C0, alpha=1.5, beta=0.5, dtype=dt)
    assert_parity(got, ref, Ar, Bc, C0, 1.5, 0.5, dt, is_tf32(name), tol, name, tc=name.startswith("tc_"))
    del A, B, Cd
    torch.cuda.empty_cache()


def test_host_mode_tasks_on_two_streams_do_not_share_staging_early(ctx):
    """host-mode tasks stage A / B / C through the context's buffers; a task submitted on
    another stream must wait until the previous host task is done with them (staging_free event).
    Two back-to-back host-mode tasks on different streams, different inputs: both results exact."""
    m, n, k = 2048, 1024, 2048          # long enough that the first GEMM is still running at the second submit
    outs, refs = [], []
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    tids = []
    for i, s in enumerate((s1, s2)):
        A = gen.matrix(gen.TAG_A, m, k, gen.DIST_I, "f32", seed=40 + i)
        B = gen.matrix(gen.TAG_B, k, n, gen.DIST_I, "f32", seed=40 + i)
        C0 = gen.matrix(gen.TAG_C, m, n, gen.DIST_I, "f32", seed=40 + i)
        Ah, Bh, Ch = (torch.from_numpy(x.copy()).pin_memory() for x in (A, B, C0))
        d = cm.make_desc(m, n, k, A=Ah, B=Bh, C_in=Ch, C_out=Ch, alpha=2.0, beta=-1.0, compute=cm.COMPUTE_TF32,
                         mem=cm.MEM_HOST, stream=s.cuda_stream, variant_hint=vid(ctx, "tc_tf32"))
        tids.append(ctx.submit(d))
        outs.append((Ah, Bh, Ch))
        rows = np.arange(0, m, 97)
        refs.append((rows, og.gemm(A[rows], B, C0[rows], alpha=2.0, beta=-1.0)))
    for t in tids:
        assert ctx.sync(t).status == 0
    for (Ah, Bh, Ch), (rows, ref) in zip(outs, refs):
        np.testing.assert_array_equal(Ch.numpy()[rows].astype(np.float64), ref)


@pytest.mark.parametrize("m,n,k,ok", [(2048, 2048, 2048, True), (1024, 1024, 1024, True), (2048, 1536, 4160, True),
                                      (128 * 148, 256, 512, True), (128 * 149, 256, 512, False),
                                      (8192, 8192, 8192, False), (32768, 32768, 32768, False),
                                      (1024, 1024, 64, False)])
def test_cluster_splitk_single_wave_eligibility(ctx, m, n, k, ok):
    """tc_*_ck is a single-wave form: eligible iff K spans >= 2 k-blocks (BF16: > 64) and the 128 x 256
    tiles fit one wave of clusters (ceil(m/128) * ceil(n/256) <= SMs); selection only, no launch."""
    buf = torch.empty(64, device="cuda", dtype=torch.float32)
    d = cm.make_desc(m, n, k, A=buf, B=buf, C_in=buf, C_out=buf, lda=k, ldb=n, ldc_in=n, ldc_out=n, alpha=1.0,
                     beta=0.5, in_dtype=cm.BF16, compute=cm.COMPUTE_BF16,
                     stream=torch.cuda.current_stream().cuda_stream)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    if m == 128 * 149 and sms > 148:
        pytest.skip("boundary case written for 148 SMs")
    assert (vid(ctx, "tc_bf16_ck") in ctx.eligible(d)) == ok


@pytest.mark.parametrize("dt", ["bf16", "f32"])
@pytest.mark.parametrize("transB", [0, 1])
@pytest.mark.parametrize("shape,beta", [((1024, 1024, 3072), 0.5), ((2048, 1536, 1000), 0.0), ((300, 520, 1000), -1.0)],
                         ids=lambda x: "x".join(map(str, x)) if isinstance(x, tuple) else str(x))
def test_unsplit_tcgen05_forms_bitwise_identical(ctx, dt, transB, shape, beta):
    """The 1-SM, CTA-pair and wide-pair forms sum every element's k in the same K = 16 (BF16) / 8
    (TF32) MMA steps into an FP32 TMEM accumulator, so their C is bitwise identical on real-valued
    inputs (only the split-K forms, which sum K ranges separately, differ) — what lets a launcher
    (tc_f32x3, the world pipeline) pick among them by shape without changing any result."""
    m, n, k = shape
    bf = dt == "bf16"
    A = device_matrix(gen.TAG_A, m, k, dtype=dt)
    B = device_matrix(gen.TAG_B, k, n, dtype=dt, transposed=bool(transB))
    C0 = device_matrix(gen.TAG_C, m, n)
    outs = {}
    for name in (("tc_bf16", "tc_bf16_2sm", "tc_bf16_2sm_w") if bf else ("tc_tf32", "tc_tf32_2sm", "tc_tf32_2sm_w")):
        Cd = C0.clone()
        d = cm.make_desc(m, n, k, A=A, B=B, C_in=Cd, C_out=Cd, ldb=k if transB else n, alpha=1.5, beta=beta,
                         in_dtype=cm.BF16 if bf else cm.F32, compute=cm.COMPUTE_BF16 if bf else cm.COMPUTE_TF32,
                         transB=transB, variant_hint=vid(ctx, name), stream=torch.cuda.current_stream().cuda_stream)
        assert ctx.run(d).status == 0
        outs[name] = Cd
    ref = next(iter(outs.values()))
    for name, o in outs.items():
        assert torch.equal(o, ref), name


def test_host_pipeline_pageable_cout_uses_copy_engine(ctx):
    """mem = HOST with a PAGEABLE C_out (no device alias): the pipeline copies C back with the copy
    engine instead of the mapped-memory copy kernel; the result equals the device path bitwise."""
    m, n, k = 1536, 776, 384
    A = gen.matrix(gen.TAG_A, m, k, dtype="bf16")
    B = gen.matrix(gen.TAG_B, k, n, dtype="bf16")
    C0 = gen.matrix(gen.TAG_C, m, n)
    Ah = torch.from_numpy(A.view(np.int16)).view(torch.bfloat16).pin_memory()
    Bh = torch.from_numpy(B.view(np.int16)).view(torch.bfloat16).pin_memory()
    Cin = torch.from_numpy(C0.copy()).pin_memory()
    Cout = torch.zeros((m, n), dtype=torch.float32)          # pageable
    assert not Cout.is_pinned()
    d = cm.make_desc(m, n, k, A=Ah, B=Bh, C_in=Cin, C_out=Cout, alpha=1.5, beta=0.5, in_dtype=cm.BF16,
                     compute=cm.COMPUTE_BF16, mem=cm.MEM_HOST, variant_hint=vid(ctx, "tc_bf16_2sm"))
    assert ctx.run(d).status == 0
    Ad, Bd, Cd = Ah.cuda(), Bh.cuda(), Cin.cuda()
    d2 = cm.make_desc(m, n, k, A=Ad, B=Bd, C_in=Cd, C_out=Cd, alpha=1.5, beta=0.5, in_dtype=cm.BF16,
                      compute=cm.COMPUTE_BF16, variant_hint=vid(ctx, "tc_bf16_2sm"),
                      stream=torch.cuda.current_stream().cuda_stream)
    assert ctx.run(d2).status == 0
    assert torch.equal(Cout, Cd.cpu())
