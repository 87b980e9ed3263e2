"""Copy-engine chain broadcast (compar_ce_export / compar_ce_import) with 3 processes sharing one GPU
(-m gpu): a gloo process group exchanges the IPC blobs and max-reduces the world samples; world-mode
row panels then receive B slab by slab along root -> 1 -> 2 (cudaMemcpyAsync from the upstream
rank's IPC-mapped buffer, GPU-side ready / consumed flag words).  Three consecutive tasks with
different B check the slab-reuse protocol; every rank's C panel must be BITWISE equal to the same
rows of the plain single-process call (each C element sums its full K in order)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

WORLD = 3
CASES = [("tc_bf16_2sm", "bf16", 1000, 1536, 768, 0, 1536, 4),
         ("tc_tf32_2sm", "f32", 700, 1280, 512, 1, 512, 3),
         ("tc_bf16", "bf16", 900, 1001, 640, 0, 1008, 4),     # N slabs not packable: one padded slab
         # the wide pair kernel: one fused launch per rank, waiting per slab on the chain's ready flags
         ("tc_bf16_2sm_w", "bf16", 1000, 2048, 640, 0, 2048, 4),
         ("tc_tf32_2sm_w", "f32", 700, 1536, 520, 1, 520, 3)]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, port, case, outdir):
    import torch.distributed as dist

    import gen
    from gen.device import fill
    from paper_2311_03543_b200 import compar as cm

    name, dt, m, n, k, tb, ldb, chunks = case
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=WORLD)
    torch.cuda.set_device(0)
    ctx = cm.Compar(bcast_chunks=chunks)

    def allgather(b):
        out = [None] * WORLD
        dist.all_gather_object(out, b)
        return out

    def red(p, _user):
        t = torch.tensor([p[0]], dtype=torch.int64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        p[0] = int(t.item())

    tdt = torch.bfloat16 if dt == "bf16" else torch.float32
    brows, bcols = (n, k) if tb else (k, n)
    ctx.ce_init(WORLD, rank, brows * ldb * (2 if dt == "bf16" else 4), allgather)
    ctx.set_reduce_hook(red)
    offs = cm.partition_rows(m, WORLD)
    r0, r1 = offs[rank], offs[rank + 1]
    mloc = r1 - r0
    names = [v for v, _ in ctx.variants()]
    sp = torch.cuda.current_stream().cuda_stream
    A = torch.empty((max(mloc, 1), k), dtype=tdt, device="cuda")
    if mloc:
        fill(A.data_ptr(), dt, mloc, k, k, gen.TAG_A, row0=r0, stream=sp)
    B = torch.zeros((brows, ldb), dtype=tdt, device="cuda") if rank == 0 else None
    kw = dict(alpha=1.5, beta=0.5, in_dtype=cm.BF16 if dt == "bf16" else cm.F32,
              compute=cm.COMPUTE_BF16 if dt == "bf16" else cm.COMPUTE_TF32, transB=tb, stream=sp,
              variant_hint=names.index(name))
    for it in range(3):                      # a different B each time: slab buffers are reused
        Cl = torch.empty((max(mloc, 1), n), dtype=torch.float32, device="cuda")
        if mloc:
            fill(Cl.data_ptr(), "f32", mloc, n, n, gen.TAG_C, row0=r0, stream=sp)
        if rank == 0:
            fill(B.data_ptr(), dt, brows, bcols, ldb, gen.TAG_B, seed=gen.SEED_DATA + it, stream=sp)
        d = cm.make_desc(m, n, k, A=A, B=B, C_in=Cl, C_out=Cl, lda=k, ldb=ldb, ldc_in=n, ldc_out=n, world=1, **kw)
        rep = ctx.run(d)
        assert rep.status == 0
        np.save(os.path.join(outdir, f"c{it}_r{rank}.npy"), Cl[:mloc].cpu().numpy())
    dist.barrier()
    ctx.terminate()
    dist.destroy_process_group()


@pytest.mark.parametrize("case", CASES, ids=[c[0] + f"-n{c[3]}-t{c[5]}" for c in CASES])
def test_ce_chain_broadcast_three_processes_bitwise(tmp_path, case):
    import torch.multiprocessing as mp

    import gen
    from gen.device import fill
    from paper_2311_03543_b200 import compar as cm

    mp.spawn(_worker, args=(_port(), case, str(tmp_path)), nprocs=WORLD, join=True)
    name, dt, m, n, k, tb, ldb, chunks = case
    tdt = torch.bfloat16 if dt == "bf16" else torch.float32
    brows, bcols = (n, k) if tb else (k, n)
    offs = cm.partition_rows(m, WORLD)
    with cm.Compar() as ctx:
        names = [v for v, _ in ctx.variants()]
        sp = torch.cuda.current_stream().cuda_stream
        A = torch.empty((m, k), dtype=tdt, device="cuda")
        fill(A.data_ptr(), dt, m, k, k, gen.TAG_A, stream=sp)
        B = torch.zeros((brows, ldb), dtype=tdt, device="cuda")
        for it in range(3):
            fill(B.data_ptr(), dt, brows, bcols, ldb, gen.TAG_B, seed=gen.SEED_DATA + it, stream=sp)
            C = torch.empty((m, n), dtype=torch.float32, device="cuda")
            fill(C.data_ptr(), "f32", m, n, n, gen.TAG_C, stream=sp)
            d = cm.make_desc(m, n, k, A=A, B=B, C_in=C, C_out=C, lda=k, ldb=ldb, ldc_in=n, ldc_out=n, alpha=1.5,
                             beta=0.5, in_dtype=cm.BF16 if dt == "bf16" else cm.F32,
                             compute=cm.COMPUTE_BF16 if dt == "bf16" else cm.COMPUTE_TF32, transB=tb, stream=sp,
                             variant_hint=names.index(name))
            assert ctx.run(d).status == 0
            ref = C.cpu().numpy()
            for r in range(WORLD):
                got = np.load(tmp_path / f"c{it}_r{r}.npy")
                np.testing.assert_array_equal(got, ref[offs[r]:offs[r + 1]])


def test_bench_world_path_shared_gpu():
    """bench.py's N > 1 path end to end (torchrun, 2 ranks, copy-engine broadcast) with both ranks on
    the one GPU (COMPAR_BENCH_SHARED_GPU=1, gloo process group): it must print one JSON line from
    rank 0 with n_gpus = 2.  A functional check only — two processes share the GPU."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, COMPAR_BENCH_SHARED_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_port()), os.path.join(root, "bench.py"), "--gpus", "2", "--steps", "2",
           "--warmup", "3", "--size", "2048", "--bcast", "ce", "--e2e-steps", "0", "--no-targets"]
    r = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    out = json.loads(lines[0])
    assert out["n_gpus"] == 2 and out["config"]["bcast"] == "ce" and out["value"] > 0


TASK_SHAPES = [(64, 64, 64), (300, 520, 256), (1000, 777, 333), (512, 1024, 512), (129, 257, 70), (2048, 256, 512)]


def _tasks_worker(rank, port, outdir):
    import torch.distributed as dist

    import gen
    from paper_2311_03543_b200 import compar as cm
    from tests._gpu_util import to_device

    world = 2
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    ctx = cm.Compar(lanes=2)
    ctx.world_init(world, rank)

    def red_n(buf, n, _user):
        t = torch.tensor([buf[i] for i in range(n)], dtype=torch.int64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        for i in range(n):
            buf[i] = int(t[i])
    ctx.set_reduce_n_hook(red_n)
    reps, tids, bufs = [], [], []
    for rnd in range(2):                     # round 0 trains the selector; round 1 is placed by dmda
        for t, (m, n, k) in enumerate(TASK_SHAPES * 4):
            A = to_device(gen.matrix(gen.TAG_A, m, k, gen.DIST_I, "f32", seed=t))
            B = to_device(gen.matrix(gen.TAG_B, k, n, gen.DIST_I, "f32", seed=t))
            C = to_device(gen.matrix(gen.TAG_C, m, n, gen.DIST_I, "f32", seed=t))
            h = 3 * (len(TASK_SHAPES) * 4 * rnd + t) + 1     # data handles: identical on both ranks
            d = cm.make_desc(m, n, k, A=A, B=B, C_in=C, C_out=C, alpha=2.0, beta=-1.0, compute=cm.COMPUTE_TF32,
                             world=cm.WORLD_TASKS, stream=torch.cuda.current_stream().cuda_stream,
                             handles=(h, h + 1, h + 2, h + 2))
            tids.append((rnd, t, ctx.submit(d)))
            bufs.append((A, B, C))
        for (r_, t, tid), (_, _, C) in zip(tids, bufs):    # collective syncs, in submission order
            r = ctx.sync(tid)
            assert r.status == 0
            if r_ == 1:
                reps.append((r.variant, r.rank, r.lane))
                if r.rank == rank:
                    np.save(os.path.join(outdir, f"t{t}.npy"), C.cpu().numpy())
        tids, bufs = [], []
    np.save(os.path.join(outdir, f"reps_r{rank}.npy"), np.array(reps))
    ctx.terminate()
    dist.destroy_process_group()


def test_task_world_two_processes_real_kernels(tmp_path):
    """NEXT-1 (task-parallel world) with two processes on the one GPU, real kernels, lanes = 2, the
    sample exchange through a gloo reduce_n hook (compar_world_init: no NCCL) and caller data
    handles (the processes' pointers differ): both ranks take identical (variant, rank, lane)
    decisions, each task runs exactly on the rank its report names, and that rank's C is bitwise
    the oracle's (integer inputs)."""
    import torch.multiprocessing as mp

    import gen
    from oracle import gemm as og

    mp.spawn(_tasks_worker, args=(_port(), str(tmp_path)), nprocs=2, join=True)
    r0, r1 = np.load(tmp_path / "reps_r0.npy"), np.load(tmp_path / "reps_r1.npy")
    bad = [(i, r0[i].tolist(), r1[i].tolist()) for i in range(len(r0)) if (r0[i] != r1[i]).any()]
    assert not bad, bad
    assert set(r0[:, 1].tolist()) == {0, 1}                  # both ranks got work
    for t, (m, n, k) in enumerate(TASK_SHAPES * 4):
        A = gen.matrix(gen.TAG_A, m, k, gen.DIST_I, "f32", seed=t)
        B = gen.matrix(gen.TAG_B, k, n, gen.DIST_I, "f32", seed=t)
        C0 = gen.matrix(gen.TAG_C, m, n, gen.DIST_I, "f32", seed=t)
        np.testing.assert_array_equal(np.load(tmp_path / f"t{t}.npy").astype(np.float64),
                                      og.gemm(A, B, C0, alpha=2.0, beta=-1.0))


def _dead_peer_worker(rank, port, outdir):
    import torch.distributed as dist

    import gen
    from gen.device import fill
    from paper_2311_03543_b200 import compar as cm

    world = 2
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    ctx = cm.Compar(bcast_chunks=2, sync_timeout_ms=2000)

    def allgather(b):
        out = [None] * world
        dist.all_gather_object(out, b)
        return out
    m = n = k = 512
    ctx.ce_init(world, rank, k * n * 2, allgather)
    names = [v for v, _ in ctx.variants()]
    sp = torch.cuda.current_stream().cuda_stream
    offs = cm.partition_rows(m, world)
    mloc = offs[rank + 1] - offs[rank]
    A = torch.empty((mloc, k), dtype=torch.bfloat16, device="cuda")
    C = torch.empty((mloc, n), dtype=torch.float32, device="cuda")
    B = torch.empty((k, n), dtype=torch.bfloat16, device="cuda")
    fill(A.data_ptr(), "bf16", mloc, k, k, gen.TAG_A, row0=offs[rank], stream=sp)
    fill(C.data_ptr(), "f32", mloc, n, n, gen.TAG_C, row0=offs[rank], stream=sp)
    fill(B.data_ptr(), "bf16", k, n, n, gen.TAG_B, stream=sp)
    d = cm.make_desc(m, n, k, A=A, B=B if rank == 0 else None, C_in=C, C_out=C, alpha=1.5, beta=0.5,
                     in_dtype=cm.BF16, compute=cm.COMPUTE_BF16, stream=sp, world=1, B_replica=B if rank else None,
                     variant_hint=names.index("tc_bf16"))   # hinted: no sample exchange with the peer
    assert ctx.run(d).status == 0                         # task 1: both ranks alive
    dist.barrier()
    if rank == 1:                                         # the peer dies without a word
        os._exit(0)
    out = {}
    s, r = ctx.sync_status(ctx.submit(d))                 # task 2: rank 1 consumed task 1's slabs
    out["t2"] = s
    t3 = ctx.submit(d)                                    # task 3 needs rank 1 to consume task 2's slabs
    import time
    t0 = time.perf_counter()
    s3, r3 = ctx.sync_status(t3)
    out["t3"], out["t3_s"] = s3, time.perf_counter() - t0
    out["t3_msg"] = cm.lib.compar_last_error(None).decode()
    try:
        ctx.submit(d)
        out["t4"] = 0
    except cm.ComparError as e:                           # sticky
        out["t4"] = e.status
    np.save(os.path.join(outdir, "dead_peer.npy"), np.array([out["t2"], out["t3"], out["t3_s"], out["t4"]]))
    with open(os.path.join(outdir, "msg.txt"), "w") as f:
        f.write(out["t3_msg"])
    os._exit(0)                                           # the comm stream is stuck on the dead peer


def test_dead_peer_wait_times_out_with_sticky_error(tmp_path):
    """R36: a rank whose peer died does not hang — the wait for the copy-engine chain (or NCCL) polls
    with sync_timeout_ms, the task fails with E_NCCL within the timeout, and every later cross-rank
    task fails with E_NCCL at submit (sticky)."""
    import torch.multiprocessing as mp

    from paper_2311_03543_b200 import compar as cm
    mp.spawn(_dead_peer_worker, args=(_port(), str(tmp_path)), nprocs=2, join=True)
    t2, t3, t3_s, t4 = np.load(tmp_path / "dead_peer.npy")
    assert t2 == cm.OK
    assert t3 == cm.E_NCCL and 1.5 < t3_s < 30, (t3, t3_s)
    assert t4 == cm.E_NCCL
    assert "timed out" in (tmp_path / "msg.txt").read_text()
