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


# ---------------------------------------------------------------- task-parallel world (NEXT-1)
def _tasks_worker(rank, world, port, lanes, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2311_03543_b200 import compar as cm
    from tests.test_dmda import Workload, cost as tcost
    ctx = cm.Compar(virtual_clock=1, lanes=lanes)
    ran = []
    cur = [None]
    for v in range(3):
        def run(desc, panel, stream, user, vns, v=v):
            ran.append(cur[0])
            vns[0] = tcost(v, desc.contents.m) + 3 * rank      # ranks measure slightly differently
            return 0
        ctx.register_variant(f"v{v}", cm.TGT_USER, run)
    ctx.comm_init(world, rank, b"\0" * 128)

    def reduce_n(buf, n, user):
        t = torch.tensor([buf[i] for i in range(n)], dtype=torch.int64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        for i in range(n):
            buf[i] = int(t[i])
    ctx.set_reduce_n_hook(reduce_n)
    wl = Workload(seed=11 + lanes, n=90)
    decisions, pending = [], []
    for i, (s, a, b, c, beta, sync) in enumerate(wl.tasks):
        cur[0] = i
        d = cm.make_desc(s, s, s, A=a, B=b, C_in=c, C_out=c, lda=s, ldb=s, ldc_in=s, ldc_out=s, alpha=1.0,
                         beta=beta, world=cm.WORLD_TASKS)
        try:
            pending.append((i, ctx.submit(d)))
        except cm.ComparError as e:           # bytes of a read span last written on two ranks (R22)
            assert e.status == cm.E_INVALID
            decisions.append((i, "refused", None, None, None, None))
        if sync or i == len(wl.tasks) - 1:
            for j, t in pending:                     # collective: same order on every rank
                r = ctx.sync(t)                      # (implicitly harvested tasks keep their reports)
                decisions.append((j, r.variant, r.mode, r.rank, r.lane, r.ns))
            ctx.sync()
            pending = []
    # a task reading two buffers last written on different ranks is refused on every rank: after a
    # full sync, three trained independent writers fill w0, w1, w2, ... (list scheduling)
    cur[0] = "extra"
    bufs = [0x7000000, 0x7100000, 0x7200000]
    kw = dict(lda=64, ldb=64, ldc_in=64, ldc_out=64, alpha=1.0, world=cm.WORLD_TASKS)
    for x in bufs:
        ctx.submit(cm.make_desc(64, 64, 64, A=0x100, B=0x200, C_out=x, **kw))
    other = bufs[1] if lanes == 1 else bufs[2]            # written on rank 1
    refused = False
    try:
        ctx.submit(cm.make_desc(64, 64, 64, A=bufs[0], B=other, C_out=0x7300000, **kw))
    except cm.ComparError as e:
        refused = e.status == cm.E_INVALID
    ok = ctx.submit(cm.make_desc(64, 64, 64, A=bufs[0], B=0x200, C_out=0x7400000, **kw))
    ctx.sync()
    ctx.terminate()
    q.put((rank, decisions, ran, refused, ok > 0))
    dist.destroy_process_group()


@pytest.mark.parametrize("lanes", [1, 2])
def test_task_world_two_ranks_matches_dmda_oracle(lanes):
    from oracle.dmda import DmdaOracle
    from tests.test_dmda import Workload, cost as tcost
    world = 2
    ctx_mp = mp.get_context("spawn")
    q = ctx_mp.Queue()
    port = _free_port()
    procs = [ctx_mp.Process(target=_tasks_worker, args=(r, world, port, lanes, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        rank, dec, ran, refused, rr = q.get(timeout=240)
        out[rank] = (dec, ran, refused, rr)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert out[0][0] == out[1][0]                       # identical reports on both ranks
    assert out[0][2] and out[1][2]                       # cross-rank read refused on both
    assert out[0][3] and out[1][3]                       # a single-rank read is accepted
    # every task ran exactly once, on the rank its report names
    wl = Workload(seed=11 + lanes, n=90)
    ran0, ran1 = set(out[0][1]), set(out[1][1])
    ran0.discard("extra")
    ran1.discard("extra")
    assert not (ran0 & ran1)
    refused_tasks = {j for (j, v, *_rest) in out[0][0] if v == "refused"}
    for (j, v, mode, rank, lane, ns) in out[0][0]:
        if v != "refused":
            assert j in (ran0 if rank == 0 else ran1)
    assert not (refused_tasks & (ran0 | ran1))
    # decisions equal the oracle's, with the owner's cost as the sample
    orc = DmdaOracle(3, nranks=world, lanes=lanes)
    exp = {}
    for i, (s, a, b, c, beta, sync) in enumerate(wl.tasks):
        reads, writes = Workload.spans(s, a, b, c, beta)
        owner = {}

        def cst(v, s=s, i=i):
            return tcost(v, s) + 3 * (exp[i][2] // lanes if i in exp else 0)
        # the sample depends on the owner rank, known only after placement: place, then fix up
        res = orc.submit(i, (s, beta != 0), [0, 1, 2], reads, writes, lambda v: 0)
        if res is None:                      # refused: a read span last written on two ranks
            exp[i] = "refused"
            if sync or i == len(wl.tasks) - 1:
                orc.sync_all()
            continue
        v, mode, w = res
        exp[i] = (v, mode, w)
        task, pv, key, pmode, warm, _, hist = orc.pending[-1]
        orc.pending[-1] = (task, pv, key, pmode, warm, tcost(v, s) + 3 * (w // lanes), hist)
        if sync or i == len(wl.tasks) - 1:
            orc.sync_all()
    got = {j: ("refused" if v == "refused" else (v, mode, rank * lanes + lane))
           for (j, v, mode, rank, lane, ns) in out[0][0]}
    assert len(got) > 40 and len(got) == len(wl.tasks)
    assert ran0 | ran1 == {j for j, g in got.items() if g != "refused"}
    for j, g in got.items():
        assert g == exp[j], j
    assert {rank for (_, v, _, rank, _, _) in out[0][0] if v != "refused"} == {0, 1}
