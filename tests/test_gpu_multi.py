"""Multi-GPU row panels (BASELINE config 4) through the driver's launch form (-m gpu).

* bench.py --gpus 2 WITHOUT torchrun (it re-executes itself as 2 ranks), both ranks on this one GPU
  (COMPAR_BENCH_SHARED_GPU=1, copy-engine broadcast, gloo): the line says n_gpus = 2 and the two
  C panels of one fresh step are BITWISE the N = 1 result (each element sums its full K in order);
* on a box with >= 2 GPUs (skipped otherwise — a skip is not a pass): 2 ranks over real NCCL —
  every receiver's B replica byte-equals root B (one slab, caller-owned replica), and the row
  panels of every built-in BF16 tensor-core variant are bitwise the single-GPU result, for the
  fused (wide kernel, flag-waiting) and the per-slab pipelines.
"""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _bench(args, env_extra):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env.update(env_extra)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


@pytest.mark.parametrize("variant", ["tc_bf16_2sm_w", "tc_bf16_2sm"])
def test_bench_gpus2_self_launch_bitwise_vs_n1(tmp_path, variant):
    common = ["--steps", "2", "--warmup", "3", "--size", "2048", "--e2e-steps", "0", "--no-targets",
              "--no-yardstick", "--no-cpu-baseline", "--variant", variant]
    one = _bench(common + ["--gpus", "1", "--dump-c", str(tmp_path / "n1")], {})
    two = _bench(common + ["--gpus", "2", "--bcast", "ce", "--dump-c", str(tmp_path / "n2")],
                 {"COMPAR_BENCH_SHARED_GPU": "1"})
    assert one["n_gpus"] == 1 and two["n_gpus"] == 2
    assert two["config"]["parallelism"] == "rowpanel2"
    c1 = np.load(tmp_path / "n1" / "c_r0.npy")
    c2 = np.concatenate([np.load(tmp_path / "n2" / f"c_r{r}.npy") for r in range(2)])
    assert c1.shape == (2048, 2048) and c2.shape == c1.shape
    np.testing.assert_array_equal(c2, c1)


# ---------------------------------------------------------------- >= 2 GPUs: real NCCL
need2 = pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs (a skip is not a pass)")


def _nccl_worker(rank, world, port, outdir):
    import torch.distributed as dist

    import gen
    from gen.device import fill
    from paper_2311_03543_b200 import compar as cm
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    sp = torch.cuda.current_stream().cuda_stream
    m, n, k = 3000, 4096, 1024
    offs = cm.partition_rows(m, world)
    r0, r1 = offs[rank], offs[rank + 1]
    res = {}
    for chunks, names in ((1, ["tc_bf16"]), (4, ["tc_bf16", "tc_bf16_2sm", "tc_bf16_2sm_w"])):
        ctx = cm.Compar(bcast_chunks=chunks)
        uid = [cm.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ctx.comm_init(world, rank, uid[0])
        vn = [v for v, _ in ctx.variants()]
        A = torch.empty((r1 - r0, k), dtype=torch.bfloat16, device="cuda")
        fill(A.data_ptr(), "bf16", r1 - r0, k, k, gen.TAG_A, row0=r0, stream=sp)
        B = torch.zeros((k, n), dtype=torch.bfloat16, device="cuda")
        if rank == 0:
            fill(B.data_ptr(), "bf16", k, n, n, gen.TAG_B, stream=sp)
        for name in names:
            C = torch.empty((r1 - r0, n), dtype=torch.float32, device="cuda")
            fill(C.data_ptr(), "f32", r1 - r0, n, n, gen.TAG_C, row0=r0, stream=sp)
            d = cm.make_desc(m, n, k, A=A, B=B if rank == 0 else None, C_in=C, C_out=C, lda=k, ldb=n, ldc_in=n,
                             ldc_out=n, alpha=1.5, beta=0.5, in_dtype=cm.BF16, compute=cm.COMPUTE_BF16, stream=sp,
                             world=1, B_replica=B if rank else None, variant_hint=vn.index(name))
            assert ctx.run(d).status == 0
            np.save(os.path.join(outdir, f"c_{chunks}_{name}_r{rank}.npy"), C.cpu().numpy())
        if chunks == 1:   # one slab, row-major B with ldb = n: the replica is B byte for byte
            np.save(os.path.join(outdir, f"b_r{rank}.npy"), B.view(torch.int16).cpu().numpy())
        ctx.terminate()
    dist.barrier()
    dist.destroy_process_group()
    return res


@need2
def test_nccl_two_gpus_replica_bytes_and_panels_bitwise(tmp_path):
    import torch.multiprocessing as mp

    import gen
    from gen.device import fill
    from paper_2311_03543_b200 import compar as cm
    world = 2
    mp.spawn(_nccl_worker, args=(world, _port(), str(tmp_path)), nprocs=world, join=True)
    np.testing.assert_array_equal(np.load(tmp_path / "b_r1.npy"), np.load(tmp_path / "b_r0.npy"))
    m, n, k = 3000, 4096, 1024
    offs = cm.partition_rows(m, world)
    with cm.Compar() as ctx:
        vn = [v for v, _ in ctx.variants()]
        sp = torch.cuda.current_stream().cuda_stream
        A = torch.empty((m, k), dtype=torch.bfloat16, device="cuda")
        B = torch.empty((k, n), dtype=torch.bfloat16, device="cuda")
        fill(A.data_ptr(), "bf16", m, k, k, gen.TAG_A, stream=sp)
        fill(B.data_ptr(), "bf16", k, n, n, gen.TAG_B, stream=sp)
        for chunks, names in ((1, ["tc_bf16"]), (4, ["tc_bf16", "tc_bf16_2sm", "tc_bf16_2sm_w"])):
            for name in names:
                C = torch.empty((m, n), dtype=torch.float32, device="cuda")
                fill(C.data_ptr(), "f32", m, n, n, gen.TAG_C, stream=sp)
                ctx.run(cm.make_desc(m, n, k, A=A, B=B, C_in=C, C_out=C, alpha=1.5, beta=0.5, in_dtype=cm.BF16,
                                     compute=cm.COMPUTE_BF16, stream=sp, variant_hint=vn.index(name)))
                ref = C.cpu().numpy()
                for r in range(world):
                    got = np.load(tmp_path / f"c_{chunks}_{name}_r{r}.npy")
                    np.testing.assert_array_equal(got, ref[offs[r]:offs[r + 1]], err_msg=f"{name} rank {r}")


@need2
def test_bench_gpus2_real_nccl_line(tmp_path):
    """The driver's form on a multi-GPU box: n_gpus = 2 and a positive broadcast time."""
    out = _bench(["--gpus", "2", "--steps", "2", "--warmup", "3", "--size", "8192", "--e2e-steps", "0",
                  "--no-targets", "--no-yardstick", "--no-cpu-baseline"], {})
    assert out["n_gpus"] == 2 and out["bcast_ms_per_step"] > 0
