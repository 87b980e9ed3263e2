"""Task-parallel world: pins of the dmda placement oracle and the C runtime's
placement decisions against it, host-only (virtual clock, one process, several lanes)."""
import random

import pytest

from oracle import selector as so
from oracle.dmda import DmdaOracle

cm = pytest.importorskip("paper_2311_03543_b200.compar")


# ---------------------------------------------------------------- oracle pins (closed forms)
def _train(o, key, cost, n=8):
    """Run `key` until model mode on one variant set, syncing so every sample is harvested."""
    for i in range(n):
        o.submit(1000 + i, key, [0], [], [], cost)
        o.sync_all()


def test_independent_tasks_round_robin_when_costs_equal():
    """Equal predicted costs c on 3 idle workers: list scheduling fills w0, w1, w2, w0, ... and
    every predicted end is c * ceil((i + 1) / 3) (ties -> lowest worker)."""
    o = DmdaOracle(1, nranks=1, lanes=3)
    _train(o, "k", lambda v: 500)
    ws = [o.submit(i, "k", [0], [], [(10 * i, 10 * i + 1)], lambda v: 500)[2] for i in range(7)]
    assert ws == [0, 1, 2, 0, 1, 2, 0]
    assert o.ready == [1500, 1000, 1000]


def test_lpt_closed_form_mixed_costs():
    """Costs 900 (key a) and 100 (key b) on 2 workers: a, b, b, ... -> the b tasks fill w1 until
    its predicted end passes 900, then the next task goes to w0."""
    o = DmdaOracle(1, nranks=1, lanes=2)
    _train(o, "a", lambda v: 900)
    _train(o, "b", lambda v: 100)
    seq = ["a"] + ["b"] * 10
    ws = [o.submit(i, k, [0], [], [(10 * i, 10 * i + 1)], lambda v: 0)[2] for i, k in enumerate(seq)]
    assert ws == [0, 1, 1, 1, 1, 1, 1, 1, 1, 1, 0]     # w1 ends 100..900; tie at 900 + 100 -> w0
    assert o.ready == [1000, 900]


def test_in_place_chain_stays_ordered_and_on_its_rank():
    """A chain of in-place tasks on one C (RAW + WAW) runs back to back: predicted ends k * c.
    On 2 ranks the chain is pinned to the rank of its first writer even when the other is idle."""
    o = DmdaOracle(1, nranks=2, lanes=1)
    _train(o, "k", lambda v: 300)
    C = (1 << 20, (1 << 20) + 4096)
    ws = [o.submit(i, "k", [0], [C], [C], lambda v: 300)[2] for i in range(4)]
    assert ws == [0, 0, 0, 0] and o.ready == [1200, 0]
    # an independent task still goes to the idle rank
    assert o.submit(9, "k", [0], [], [(0, 8)], lambda v: 300)[2] == 1


def test_reads_from_two_ranks_are_refused():
    o = DmdaOracle(1, nranks=2, lanes=1)
    _train(o, "k", lambda v: 300)
    X, Y = (0, 64), (64, 128)
    assert o.submit(1, "k", [0], [], [X], lambda v: 300)[2] == 0
    assert o.submit(2, "k", [0], [], [Y], lambda v: 300)[2] == 1          # rank 0 busy -> rank 1
    assert o.submit(3, "k", [0], [X, Y], [(500, 600)], lambda v: 300) is None
    o.sync_all()                                                      # full sync forgets residency
    assert o.submit(4, "k", [0], [X, Y], [(500, 600)], lambda v: 300)[2] == 0


def test_split_writers_of_one_read_span_are_refused():
    """C rows [0, 500) written on rank 0 and rows [500, 1000) on rank 1 — a task
    reading all of C has bytes whose latest writers ran on two ranks: refused, although the single
    LATEST writer alone would pin it to rank 1.  A later writer covering the whole span re-pins it."""
    o = DmdaOracle(1, nranks=2, lanes=1)
    _train(o, "k", lambda v: 300)
    C = (0, 1000)
    assert o.submit(1, "k", [0], [], [(0, 500)], lambda v: 300)[2] == 0
    assert o.submit(2, "k", [0], [], [(500, 1000)], lambda v: 300)[2] == 1
    assert o.submit(3, "k", [0], [C], [(2000, 2100)], lambda v: 300) is None
    # one buffer written whole on rank 0, then its first half rewritten on rank 1: refused too
    o.sync_all()
    assert o.submit(4, "k", [0], [], [C], lambda v: 300)[2] == 0
    assert o.submit(5, "k", [0], [], [(3000, 3100)], lambda v: 300)[2] == 1
    assert o.submit(6, "k", [0], [(3000, 3100)], [(0, 500)], lambda v: 300)[2] == 1
    assert o.submit(7, "k", [0], [C], [(4000, 4100)], lambda v: 300) is None
    # ... but a whole-span rewrite on rank 1 makes every byte's latest writer rank 1
    assert o.submit(8, "k", [0], [(3000, 3100)], [C], lambda v: 300)[2] == 1
    assert o.submit(9, "k", [0], [C], [(5000, 5100)], lambda v: 300)[2] == 1


def test_runtime_refuses_split_writers_like_the_oracle():
    """The same split-writer stream through the C runtime (2 ranks, virtual clock, world_init)."""
    ctx = cm.Compar(virtual_clock=1)
    ctx.register_variant("v", cm.TGT_USER, lambda desc, panel, stream, user, vns: vns.__setitem__(0, 300) or 0)
    ctx.world_init(2, 0)
    ctx.set_reduce_n_hook(lambda buf, n, user: None)      # this process plays both ranks' samples
    kw = dict(lda=1, ldb=1, ldc_in=1, ldc_out=1, alpha=1.0, world=cm.WORLD_TASKS)

    def sub(c_out, n, beta=0.0, c_in=None):          # a 1 x n task: C spans n * 4 bytes
        return ctx.submit(cm.make_desc(1, n, 1, A=0x20, B=0x10, C_in=c_in, C_out=c_out, beta=beta,
                                       lda=1, ldb=n, ldc_in=n, ldc_out=n, alpha=1.0, world=cm.WORLD_TASKS))
    for n in (250, 500):                                 # train both keys: calibration -> model mode
        for _ in range(6):
            ctx.sync(sub(0x30000, n))
    ctx.sync()
    t1 = sub(0x1000, 250)                                # bytes [0, 1000) of C: rank 0 (both idle)
    t2 = ctx.submit(cm.make_desc(1, 250, 1, A=0x20, B=0x10, C_out=0x1000 + 1000, lda=1, ldb=250, ldc_in=250,
                                 ldc_out=250, alpha=1.0, world=cm.WORLD_TASKS))   # [1000, 2000): rank 1
    with pytest.raises(cm.ComparError) as e:             # reads all of C: halves last written on 2 ranks
        sub(0x5000, 500, beta=0.5, c_in=0x1000)
    assert e.value.status == cm.E_INVALID
    assert (ctx.sync(t1).rank, ctx.sync(t2).rank) == (0, 1)
    ctx.sync()
    ctx.terminate()


def test_war_across_ranks_needs_no_order_but_same_rank_does():
    o = DmdaOracle(1, nranks=2, lanes=2)
    _train(o, "k", lambda v: 100)
    X = (0, 64)
    assert o.submit(1, "k", [0], [X], [(100, 164)], lambda v: 100)[2] == 0     # reads X on w0
    # writer of X: w1 (rank 0) would have to wait for the reader (est 100); rank 1 is free at 0
    assert o.submit(2, "k", [0], [], [X], lambda v: 100)[2] == 2
    assert o.ready == [100, 0, 100, 0]


# ---------------------------------------------------------------- C runtime == oracle
class Workload:
    """Random in-place / out-of-place task stream over a small buffer pool (fake addresses)."""

    SIZES = [64, 128, 256]

    def __init__(self, seed, n=120):
        rnd = random.Random(seed)
        self.tasks = []
        for i in range(n):
            s = rnd.choice(self.SIZES)
            a = 0x10000000 * (1 + rnd.randrange(3))
            b = 0x40000000 + 0x10000000 * rnd.randrange(2)
            c = 0x80000000 + 0x10000000 * rnd.randrange(4)
            beta = rnd.choice([0.0, 0.5])
            sync = rnd.random() < 0.08
            self.tasks.append((s, a, b, c, beta, sync))

    @staticmethod
    def spans(s, a, b, c, beta):
        nb = ((s - 1) * s + s) * 4
        reads = [(a, a + nb), (b, b + nb)] + ([(c, c + nb)] if beta else [])
        return reads, [(c, c + nb)]


def cost(v, s):
    return [40 * s + 1000, 25 * s + 4000, 60 * s][v]


@pytest.mark.parametrize("lanes", [1, 3])
def test_runtime_placement_matches_oracle(lanes):
    ctx = cm.Compar(virtual_clock=1, lanes=lanes)
    for v in range(3):
        def run(desc, panel, stream, user, vns, v=v):
            vns[0] = cost(v, desc.contents.m)
            return 0
        ctx.register_variant(f"v{v}", cm.TGT_USER, run)
    orc = DmdaOracle(3, nranks=1, lanes=lanes)
    wl = Workload(seed=lanes)
    pending, checked = [], []
    for i, (s, a, b, c, beta, sync) in enumerate(wl.tasks):
        d = cm.make_desc(s, s, s, A=a, B=b, C_in=c, C_out=c, lda=s, ldb=s, ldc_in=s, ldc_out=s, alpha=1.0,
                         beta=beta, world=cm.WORLD_TASKS)
        t = ctx.submit(d)
        reads, writes = wl.spans(s, a, b, c, beta)
        exp = orc.submit(t, (s, beta != 0), [0, 1, 2], reads, writes, lambda v: cost(v, s))
        pending.append((t, exp))
        if sync or i == len(wl.tasks) - 1:
            reps = {}
            for tt, _ in pending:          # (tasks harvested by a decision keep their reports)
                reps[tt] = ctx.sync(tt)
            ctx.sync()
            orc.sync_all()
            for tt, (v, mode, w) in pending:
                if tt in reps:
                    r = reps[tt]
                    assert (r.variant, r.mode, r.rank * lanes + r.lane) == (v, mode, w), (i, tt)
                    checked.append((mode, w))
            pending = []
    ctx.terminate()
    assert len(checked) > 60
    assert {w for _, w in checked} == set(range(lanes))
    assert {so.MODE_CALIB, so.MODE_MODEL} <= {m for m, _ in checked}
