"""Exact-integer (bitwise) parity of the persistent tcgen05 variants on grids where every CTA (or
CTA pair) runs several tiles (-m gpu).

SURVEY §8(c) "Exact integers" pin: inputs in {-2..2}, alpha = 2, beta = -1; every partial sum is
an exact integer below 2^24 for every K <= 2^21, so EVERY variant must equal the FP64 oracle
bitwise, whatever its summation order.  The small-shape integer cases (test_gpu_parity.py) never
leave a CTA's first tile; these shapes exercise what the bench path actually runs: tile-ring wrap,
the scheduler counter re-arm between launches, the wide kernel's delayed half-1 schedule on a
CTA's 2nd+ tile, and the pair kernels' epilogue overlapping the next tile's mainloop.

* 4096 x 5120 x 1000 compared in FULL (wide pair: 160 tiles on 74 clusters; pair: 320; 1-SM: 640);
* the BASELINE full sizes in the bench launch configuration (8192^3, 32768^3, 65536 x 256 x 4096)
  compared bitwise on full rows (all column tiles) and a sampled sub-block (many row tiles).
"""
import numpy as np
import pytest

import gen
from oracle import gemm as og

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from gen.device import device_matrix  # noqa: E402

cm = pytest.importorskip("paper_2311_03543_b200.compar")

PERSISTENT = ["tc_tf32", "tc_bf16", "tc_tf32_2sm", "tc_bf16_2sm", "tc_tf32_2sm_w", "tc_bf16_2sm_w"]
ALPHA, BETA = 2.0, -1.0
I = gen.DIST_I


@pytest.fixture(scope="module")
def ctx():
    c = cm.Compar()
    yield c
    c.terminate()


def vid(ctx, name):
    return [n for n, _ in ctx.variants()].index(name)


def launch(ctx, name, m, n, k, transB=0):
    bf = "bf16" in name
    dt = "bf16" if bf else "f32"
    A = device_matrix(gen.TAG_A, m, k, I, dtype=dt)
    B = device_matrix(gen.TAG_B, k, n, I, dtype=dt, transposed=bool(transB))
    Cd = device_matrix(gen.TAG_C, m, n, I)
    d = cm.make_desc(m, n, k, A=A, B=B, C_in=Cd, C_out=Cd, ldb=k if transB else n, alpha=ALPHA, beta=BETA,
                     in_dtype=cm.BF16 if bf else cm.F32, compute=cm.COMPUTE_BF16 if bf else cm.COMPUTE_TF32,
                     transB=transB, variant_hint=vid(ctx, name), stream=torch.cuda.current_stream().cuda_stream)
    r = ctx.run(d)
    assert r.status == 0 and r.variant == vid(ctx, name)
    del A, B
    return Cd


_REF = {}


def full_ref(m, n, k):
    """Integer inputs are exact in FP32 and BF16 alike, so one oracle run serves every variant."""
    if (m, n, k) not in _REF:
        A = gen.matrix(gen.TAG_A, m, k, I, "f32")
        B = gen.matrix(gen.TAG_B, k, n, I, "f32")
        C0 = gen.matrix(gen.TAG_C, m, n, I, "f32")
        _REF[(m, n, k)] = og.gemm(A, B, C0, alpha=ALPHA, beta=BETA)
    return _REF[(m, n, k)]


@pytest.mark.parametrize("transB", [0, 1])
@pytest.mark.parametrize("name", PERSISTENT)
def test_multitile_full_compare(ctx, name, transB):
    m, n, k = 4096, 5120, 1000
    Cd = launch(ctx, name, m, n, k, transB)
    got = Cd.double().cpu().numpy()
    np.testing.assert_array_equal(got, full_ref(m, n, k))


@pytest.mark.parametrize("transB", [0, 1])
@pytest.mark.parametrize("shape", [(4096, 5120, 1000), (1000, 1200, 776)], ids=["128-tiles", "64-tiles"])
@pytest.mark.parametrize("name", ["tma_f32", "simt_f32"])
def test_ffma_multiwave_full_compare(ctx, name, shape, transB):
    """The FFMA variants over several waves of CTAs, bitwise: 4096 x 5120 x 1000 runs tma_f32's
    128-tiles (1280 tiles, 8.6 waves; 32 k-blocks with a ragged last one, so the 4-stage ring wraps
    and the register fragments read one k ahead cross every stage boundary), 1000 x 1200 x 776 its
    64-tiles (a grid of <= 3/4 of the SMs in 128-tiles; K = 776 keeps the rows 16-byte aligned, as
    TMA requires)."""
    m, n, k = shape
    got = launch(ctx, name, m, n, k, transB).double().cpu().numpy()
    np.testing.assert_array_equal(got, full_ref(m, n, k))


def test_multitile_full_compare_splitk(ctx):
    """The split-K variants over many (tile, k-range) work items and the cluster split-K variants over
    many clusters (several waves): bitwise too (partials summed in split order, every partial an
    exact integer)."""
    m, n, k = 2048, 1536, 4160
    ref = full_ref(m, n, k)
    for name in ("tc_tf32_sk", "tc_bf16_sk", "tc_tf32_ck", "tc_bf16_ck"):
        got = launch(ctx, name, m, n, k).double().cpu().numpy()
        np.testing.assert_array_equal(got, ref, err_msg=name)


def sample_rows(m, tile=256, extra=16, seed=3):
    """Rows at the first/last row of the first, second, middle and last tiles, plus random rows."""
    rng = np.random.default_rng(seed)
    fixed = [0, 1, tile - 1, tile, 2 * tile - 1, m // 2 - 1, m // 2, m - tile - 1, m - tile, m - 1]
    return np.unique(np.clip(np.concatenate([fixed, rng.integers(0, m, extra)]), 0, m - 1)).astype(np.int64)


@pytest.mark.parametrize("name,shape", [(nm, (8192, 8192, 8192)) for nm in PERSISTENT] +
                         [(nm, (65536, 256, 4096)) for nm in PERSISTENT] +
                         [("tc_bf16", (32768, 32768, 32768)), ("tc_bf16_2sm", (32768, 32768, 32768)),
                          ("tc_bf16_2sm_w", (32768, 32768, 32768)), ("tc_tf32_2sm_w", (32768, 32768, 32768))],
                         ids=lambda x: x if isinstance(x, str) else "x".join(map(str, x)))
def test_full_size_exact_sampled(ctx, name, shape):
    """Bench-size launches (many tiles per CTA), bitwise on sampled entries against the oracle."""
    m, n, k = shape
    Cd = launch(ctx, name, m, n, k)
    rows = sample_rows(m)
    rng = np.random.default_rng(9)
    Ar = gen.matrix_rows(gen.TAG_A, rows, k, I, "f32")
    if n * k <= 8192 * 8192:   # full rows: every column tile of these row tiles
        Bf = gen.matrix(gen.TAG_B, k, n, I, "f32")
        ref = og.gemm(Ar, Bf, gen.matrix_rows(gen.TAG_C, rows, n, I), alpha=ALPHA, beta=BETA)
        got = Cd[torch.as_tensor(rows, device="cuda")].double().cpu().numpy()
        np.testing.assert_array_equal(got, ref)
    # sampled sub-block over many row and column tiles
    r2 = np.unique(np.concatenate([rows, rng.integers(0, m, 48)])).astype(np.int64)
    cols = np.unique(np.concatenate([[0, 255, 256, 511, 512, n - 1], rng.integers(0, n, 40)]).clip(0, n - 1))
    cols = cols.astype(np.int64)
    ref2 = og.gemm(gen.matrix_rows(gen.TAG_A, r2, k, I, "f32"), gen.matrix_cols(gen.TAG_B, k, cols, I, "f32"),
                   gen.matrix_entries(gen.TAG_C, r2, cols, I), alpha=ALPHA, beta=BETA)
    got2 = Cd[torch.as_tensor(r2, device="cuda")][:, torch.as_tensor(cols, device="cuda")].double().cpu().numpy()
    np.testing.assert_array_equal(got2, ref2)
    del Cd
    torch.cuda.empty_cache()


# ---- pair-kernel schedule forms (tc_gemm_2sm_mc.cu): single-wave (5 stages, two staging buffers),
# deep ring (multi-wave: 6 stages, one buffer), even waves (fewest pairs with as many waves), and the
# last tile's C_in chunks staged in the drained ring — all bitwise against the oracle ----

@pytest.mark.parametrize("name", ["tc_bf16_2sm", "tc_tf32_2sm"])
@pytest.mark.parametrize("shape", [(2048, 2048, 1000), (1800, 2000, 776), (9000, 2304, 520)],
                         ids=lambda s: "x".join(map(str, s)))
def test_pair_schedule_forms_exact(ctx, name, shape):
    """64 pair tiles (single wave), the same ragged, and 36 x 9 = 324 tiles (deep ring, even waves:
    5 waves on 65 pairs, last tile staged in the ring)."""
    m, n, k = shape
    got = launch(ctx, name, m, n, k).double().cpu().numpy()
    np.testing.assert_array_equal(got, full_ref(m, n, k))


@pytest.mark.parametrize("name", ["tc_bf16_2sm", "tc_tf32_2sm"])
def test_pair_deep_ring_beta0_exact(ctx, name):
    """beta = 0 on the deep-ring form (C_in never read, stores drain through one staging buffer)."""
    m, n, k = 9000, 2304, 520
    bf = "bf16" in name
    dt = "bf16" if bf else "f32"
    A = device_matrix(gen.TAG_A, m, k, I, dtype=dt)
    B = device_matrix(gen.TAG_B, k, n, I, dtype=dt)
    Cd = torch.full((m, n), float("nan"), device="cuda")
    d = cm.make_desc(m, n, k, A=A, B=B, C_in=Cd, C_out=Cd, alpha=ALPHA, beta=0.0,
                     in_dtype=cm.BF16 if bf else cm.F32, compute=cm.COMPUTE_BF16 if bf else cm.COMPUTE_TF32,
                     variant_hint=vid(ctx, name), stream=torch.cuda.current_stream().cuda_stream)
    assert ctx.run(d).status == 0
    ref = og.gemm(gen.matrix(gen.TAG_A, m, k, I, "f32"), gen.matrix(gen.TAG_B, k, n, I, "f32"), alpha=ALPHA)
    np.testing.assert_array_equal(Cd.double().cpu().numpy(), ref)
