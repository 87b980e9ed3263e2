"""Task-parallel world on the GPU (-m gpu): several lanes (library streams)
on one B200, real kernels.  Independent tasks land on different lanes and stay correct; in-place
chains on one buffer are ordered by the buffer dependency tracking even when the placer spreads
the surrounding work over lanes (checked bitwise on integer data against the FP64 oracle)."""
import numpy as np
import pytest

import gen
from gen.device import device_matrix
from oracle import gemm as og

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from tests._gpu_util import to_device, to_host_f64  # noqa: E402

cm = pytest.importorskip("paper_2311_03543_b200.compar")


def _desc(A, B, C, beta, compute=None, alpha=2.0):
    m, k = A.shape
    n = B.shape[1]
    return cm.make_desc(m, n, k, A=A, B=B, C_in=C, C_out=C, alpha=alpha, beta=beta,
                        compute=cm.COMPUTE_TF32 if compute is None else compute, world=cm.WORLD_TASKS,
                        stream=torch.cuda.current_stream().cuda_stream)


@pytest.mark.parametrize("lanes", [1, 3])
def test_independent_and_chained_tasks(lanes):
    rng = np.random.default_rng(5)
    ctx = cm.Compar(lanes=lanes)
    # 6 independent problems of mixed sizes, each run 5 times in place (a chain per buffer)
    probs = []
    for i, (m, n, k) in enumerate([(256, 256, 256), (512, 384, 128), (130, 70, 300), (1024, 1024, 512),
                                   (64, 64, 64), (700, 300, 260)]):
        A = gen.matrix(gen.TAG_A, m, k, gen.DIST_I, "f32", seed=100 + i)
        B = gen.matrix(gen.TAG_B, k, n, gen.DIST_I, "f32", seed=100 + i)
        C = gen.matrix(gen.TAG_C, m, n, gen.DIST_I, "f32", seed=100 + i).astype(np.float64)
        probs.append([to_device(A), to_device(B), to_device(C.astype(np.float32)), A, B, C])
    order = [i for i in range(len(probs)) for _ in range(5)]
    rng.shuffle(order)
    lanes_used = set()
    for rnd in range(3):                     # round 0 calibrates; rounds 1-2 run in model mode
        tids = []
        for i in order:
            Ad, Bd, Cd, A, B, C = probs[i]
            beta = -1.0
            tids.append(ctx.submit(_desc(Ad, Bd, Cd, beta)))
            probs[i][5] = og.gemm(A, B, probs[i][5], alpha=2.0, beta=beta, dtype="f32")
        for t in tids:          # implicitly harvested tasks keep their reports until synced
            r = ctx.sync(t)
            lanes_used.add(r.lane)
            assert r.status == 0 and r.rank == 0
        ctx.sync()
        torch.cuda.synchronize()
        for Ad, Bd, Cd, A, B, C in probs:
            np.testing.assert_array_equal(to_host_f64(Cd), C)
    assert lanes_used == set(range(lanes))
    ctx.terminate()


def test_lanes_run_concurrently():
    """Eight independent 2048^3 TF32 tasks: with 4 lanes the placer spreads them and the stream
    finishes no slower than with 1 lane (same kernels; concurrency may only help)."""
    import time
    m = 2048
    A = [device_matrix(gen.TAG_A, m, m, seed=s) for s in range(8)]
    B = device_matrix(gen.TAG_B, m, m)
    Cs = [torch.zeros(m, m, device="cuda") for _ in range(8)]
    times = {}
    for lanes in (1, 4):
        ctx = cm.Compar(lanes=lanes)
        for rnd in range(4):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for i in range(8):
                ctx.submit(_desc(A[i], B, Cs[i], 0.0, alpha=1.0))
            ctx.sync()
            torch.cuda.synchronize()
            times[lanes] = time.perf_counter() - t0
        ctx.terminate()
    assert times[4] <= times[1] * 1.10, times
