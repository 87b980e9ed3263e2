"""The sort interface on the GPU (-m gpu): both sm_100a variants against the
oracle (bit-exact: the sorted order is unique as bit patterns under IEEE totalOrder), edge cases,
and the history selector over the sort variants."""
import numpy as np
import pytest

from oracle import sort as osort

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

cm = pytest.importorskip("paper_2311_03543_b200.compar")

KT = {osort.KEY_U32: (np.uint32, torch.int32), osort.KEY_I32: (np.int32, torch.int32),
      osort.KEY_F32: (np.float32, torch.float32)}


@pytest.fixture(scope="module")
def ctx():
    c = cm.Compar()
    yield c
    c.terminate()


def vid(ctx, name):
    return [n for n, _ in ctx.variants()].index(name)


def keys_for(kt, n, dist, seed):
    rng = np.random.default_rng(seed)
    if dist == "dup":
        x = rng.integers(0, 7, n).astype(np.uint32)
    elif dist == "sorted":
        x = np.sort(rng.integers(0, 2 ** 32, n, dtype=np.uint64).astype(np.uint32))
    elif dist == "reverse":
        x = np.sort(rng.integers(0, 2 ** 32, n, dtype=np.uint64).astype(np.uint32))[::-1].copy()
    else:
        x = rng.integers(0, 2 ** 32, n, dtype=np.uint64).astype(np.uint32)
    if kt == osort.KEY_F32 and dist == "special":
        sp = np.array([0x7FC00000, 0xFFC00000, 0x7F800000, 0xFF800000, 0x0, 0x80000000, 0x1, 0x80000001],
                      dtype=np.uint32)
        x[rng.integers(0, n, max(1, n // 5))] = rng.choice(sp, max(1, n // 5))
    return x.view(KT[kt][0])


def run_sort(ctx, name, keys_np, kt):
    t = torch.from_numpy(keys_np.view(np.int32) if kt != osort.KEY_F32 else keys_np).cuda()
    r = ctx.sort(t, key_type=kt, variant_hint=vid(ctx, name), stream=torch.cuda.current_stream().cuda_stream)
    got = t.cpu().numpy().view(KT[kt][0])
    return r, got


SIZES = [2, 3, 17, 1000, 4096, 8191, 8192, 8193, 16384]


@pytest.mark.parametrize("name", ["sort_radix", "sort_bitonic"])
@pytest.mark.parametrize("kt", [osort.KEY_U32, osort.KEY_I32, osort.KEY_F32])
@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("dist", ["uniform", "dup", "special", "sorted", "reverse"])
def test_sort_parity_small(ctx, name, kt, n, dist):
    x = keys_for(kt, n, dist, seed=n + kt)
    r, got = run_sort(ctx, name, x, kt)
    assert r.status == 0 and r.variant == vid(ctx, name)
    np.testing.assert_array_equal(got.view(np.uint32), osort.sort(x, kt).view(np.uint32))


@pytest.mark.parametrize("kt", [osort.KEY_U32, osort.KEY_F32])
@pytest.mark.parametrize("n", [100000, 1 << 20, 3_000_001, 1 << 26])
def test_radix_parity_large(ctx, kt, n):
    x = keys_for(kt, n, "special" if kt == osort.KEY_F32 else "uniform", seed=7)
    r, got = run_sort(ctx, "sort_radix", x, kt)
    assert r.status == 0
    np.testing.assert_array_equal(got.view(np.uint32), osort.sort(x, kt).view(np.uint32))


def test_noop_and_validation(ctx):
    t = torch.tensor([3.0], device="cuda")
    assert ctx.sort(t).mode == cm.MODE_NOOP and t.item() == 3.0
    assert ctx.sort(torch.empty(0, device="cuda")).mode == cm.MODE_NOOP
    with pytest.raises(cm.ComparError):                       # bitonic cannot take n > 16384
        ctx.sort(torch.zeros(20000, device="cuda"), variant_hint=vid(ctx, "sort_bitonic"))
    with pytest.raises(cm.ComparError):                       # a GEMM variant is not a sort variant
        ctx.sort(torch.zeros(100, device="cuda"), variant_hint=vid(ctx, "tc_bf16"))


def test_selector_over_sort_variants(ctx):
    """Unseen key: blocked calibration over the eligible sort variants, then model mode picks the
    measured argmin; n > 16384 leaves only the radix sort."""
    for n, expect_elig in ((4096, {"sort_radix", "sort_bitonic"}), (100000, {"sort_radix"})):
        x = keys_for(osort.KEY_F32, n, "uniform", seed=1)
        t = torch.from_numpy(x).cuda()
        reps = []
        for _ in range(4 * len(expect_elig) + 3):
            t.copy_(torch.from_numpy(x))
            reps.append(ctx.sort(t, stream=torch.cuda.current_stream().cuda_stream))
        names = [nm for nm, _ in ctx.variants()]
        assert {names[r.variant] for r in reps[:4 * len(expect_elig)]} == expect_elig
        assert reps[-1].mode == cm.MODE_MODEL
        # the model pick is the calibrated argmin of the per-variant means of the timed samples
        cal = {}
        for r in reps[:4 * len(expect_elig)]:
            if r.mode == cm.MODE_CALIB:
                cal.setdefault(names[r.variant], []).append(r.ns)
        means = {k: sum(v) / len(v) for k, v in cal.items()}
        assert names[reps[4 * len(expect_elig)].variant] == min(means, key=means.get)
        np.testing.assert_array_equal(t.cpu().numpy().view(np.uint32), osort.sort(x).view(np.uint32))
