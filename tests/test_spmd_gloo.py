"""SPMD (one process per GPU) host logic on CPU with world_size 2 over gloo (-m "not gpu").

Runs the runtime in virtual-clock mode in two processes: each rank owns the row panel
compar_partition_rows(m, 2)[rank] of every world-mode task, reports a synthetic cost that
depends on its rank and panel, and the per-task sample is max-reduced across ranks through the
reduce hook (gloo all_reduce MAX) — the same role the NCCL all-reduce plays on GPUs.  Checks:
panel rows follow the a4 formula, every rank takes IDENTICAL decisions, and those decisions
equal the selector oracle fed with the max-over-ranks samples.
"""
import os
import socket

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from oracle import selector as so  # noqa: E402
from oracle.partition import partition_rows  # noqa: E402

SIZES = [1000, 4096, 300, 4096, 1000, 129, 4096, 300, 1000, 129] * 4


def cost(v, rank, rows):
    return [rows * 10 + 7 * rank + 1, 3000 + rows * 3 + 400 * rank][v]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2311_03543_b200 import compar as cm
    ctx = cm.Compar(virtual_clock=1)
    seen_rows = []

    def make(v):
        def run(desc, panel, stream, user, vns):
            rows = panel.contents.rows
            seen_rows.append((v, panel.contents.row0, rows))
            vns[0] = cost(v, rank, rows)
            return 0
        return run
    for v in range(2):
        ctx.register_variant(f"v{v}", cm.TGT_USER, make(v))
    ctx.comm_init(world, rank, b"\0" * 128)

    def reduce(ptr, user):
        t = torch.tensor([ptr[0]], dtype=torch.int64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ptr[0] = int(t.item())
    ctx.set_reduce_hook(reduce)
    decisions = []
    for m in SIZES:
        d = cm.make_desc(m, 64, 64, lda=64, ldb=64, ldc_in=64, ldc_out=64, alpha=1.0, beta=0.5, world=1)
        r = ctx.run(d)
        decisions.append((r.variant, r.mode, r.ns))
    ctx.terminate()
    q.put((rank, decisions, seen_rows))
    dist.destroy_process_group()


def test_spmd_world2_rank_consistent_decisions():
    world = 2
    ctx_mp = mp.get_context("spawn")
    q = ctx_mp.Queue()
    port = _free_port()
    procs = [ctx_mp.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        rank, dec, rows = q.get(timeout=240)
        out[rank] = (dec, rows)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # identical decisions and identical (max-reduced) samples on every rank
    assert out[0][0] == out[1][0]
    # panels follow the a4 formula
    for rank in range(world):
        rows = out[rank][1]
        for (v, row0, nrows), m in zip(rows, SIZES):
            offs = partition_rows(m, world)
            assert (row0, nrows) == (offs[rank], offs[rank + 1] - offs[rank])
    # and equal the selector oracle fed with max-over-ranks costs
    orc = so.SelectorOracle(2, blocked=True)      # the runtime's default calibration order (R19)
    for m, (v, mode, ns) in zip(SIZES, out[0][0]):
        offs = partition_rows(m, world)
        key = offs[1] - offs[0]
        ev, emode = orc.decide(key, [0, 1])
        warm = orc.commit(ev, key, emode)
        sample = max(cost(ev, r, offs[r + 1] - offs[r]) for r in range(world))
        orc.harvest(ev, key, emode, warm, sample)
        assert (v, mode) == (ev, emode)
        assert ns == sample
