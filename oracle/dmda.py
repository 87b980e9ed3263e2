"""Task-level placement oracle — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference legs may import it;
the product path never does.  Shares no code with the C runtime (paper_2311_03543_b200/csrc/
runtime/dmda.cpp); it is written from the scheduling rule it implements:

* StarPU "handles the mapping, scheduling, and data transfers required for
  executing these tasks";
* SPEC S:326-330 (SchedulerDecision): "chosen = argmin over schedulable (variant, worker) of
  ready + exec + transfer; ties broken by lowest variant index then lowest worker index";
* SPEC S:307-311 (DataHandle): "writers order after all earlier-submitted accessors of the
  handle (sequential consistency per handle in submission order)";
* DESIGN.md readings R20-R23: workers are (rank, lane) pairs w = rank * lanes + lane; ready[w] is
  the predicted end of the last task placed on w (reset by a full sync); exec = the variant's
  measured mean for the key (integer division of the integer sums), else 0; a task that reads a
  range whose bytes were last written on rank r may only run on rank r (no inter-rank transfer:
  cost infinite), and a range whose bytes were last written on two ranks cannot be read at all;
  RAW / WAR / WAW on the same rank delay the start to the earlier task's predicted end; with
  lanes > 1, model-mode executions are not samples.

The variant decision itself is the history selector (oracle/selector.py, steps 1-7).
"""
from dataclasses import dataclass, field

from oracle.selector import MODE_CALIB, MODE_MODEL, MODE_WARMUP, SelectorOracle


def _overlap(a, b):
    return a[0] < b[1] and b[0] < a[1] and a[0] < a[1] and b[0] < b[1]


@dataclass
class DmdaOracle:
    n_variants: int
    nranks: int = 1
    lanes: int = 1
    blocked: bool = True
    prune_pct: int = 150       # the runtime's default (R32)
    sel: SelectorOracle = None
    ready: list = field(default_factory=list)
    live: list = field(default_factory=list)      # (task, w, end, span, write)
    pending: list = field(default_factory=list)   # (task, v, key, mode, warm, ns, history)

    def __post_init__(self):
        self.sel = SelectorOracle(self.n_variants, blocked=self.blocked, prune_pct=self.prune_pct)
        self.reset_workers()

    def reset_workers(self):
        self.ready = [0] * (self.nranks * self.lanes)
        self.live = []

    def rank_of(self, w):
        return w // self.lanes

    # ---- history bookkeeping (step 6 / 7)
    def _harvest(self, pred):
        keep = []
        for p in self.pending:                    # task-id order
            task, v, key, mode, warm, ns, hist = p
            if pred(p):
                if hist:
                    self.sel.harvest(v, key, mode, warm, ns)
            else:
                keep.append(p)
        self.pending = keep

    def _calibrating(self, key, eligible):
        return self.sel.calibrating(key, eligible)

    # ---- placement (SPEC S:330 with the R20-R23 readings)
    def place(self, reads, writes, exec_ns):
        # Residency (R22): every byte of a read span lives on the rank of ITS latest writer.  Cut
        # the span at every writer boundary into elementary intervals; each interval's latest
        # overlapping writer names its rank; all ranks met must agree, else nowhere may read it.
        pin = None
        for s in reads:
            writers = [(task, w, span) for (task, w, end, span, write) in self.live if write and _overlap(s, span)]
            cuts = sorted({s[0], s[1]} | {x for (_, _, sp) in writers for x in sp if s[0] < x < s[1]})
            for lo, hi in zip(cuts, cuts[1:]):
                over = [(task, w) for (task, w, sp) in writers if _overlap((lo, hi), sp)]
                if not over:
                    continue
                r = self.rank_of(max(over)[1])
                if pin is not None and pin != r:
                    return None
                pin = r
        best = None
        for w in range(self.nranks * self.lanes):
            if pin is not None and self.rank_of(w) != pin:
                continue
            est = self.ready[w]
            for (task, lw, end, span, write) in self.live:
                if self.rank_of(lw) != self.rank_of(w):
                    continue
                raw = write and any(_overlap(s, span) for s in reads)
                wx = any(_overlap(s, span) for s in writes)
                if raw or wx:
                    est = max(est, end)
            e = est + exec_ns
            if best is None or e < best[1]:
                best = (w, e)
        return best

    def submit(self, task, key, eligible, reads, writes, cost):
        """One task: returns (variant, mode, worker) or None (no worker may run it)."""
        # step 6 (and R32: pruning reads the key's best mean, so with pruning on every decision
        # harvests the key's pending samples first)
        if self.prune_pct > 0 or not self._calibrating(key, eligible):
            self._harvest(lambda p: p[2] == key)
        v, mode = self.sel.decide(key, eligible)
        r = self.sel.rec(v, key)
        exec_ns = r.sum_ns // r.count if r.count else 0
        pl = self.place(reads, writes, exec_ns)
        if pl is None:
            return None
        w, end = pl
        warm = self.sel.commit(v, key, mode)
        self.ready[w] = end
        for s in reads:
            self.live.append((task, w, end, s, False))
        for s in writes:
            self.live.append((task, w, end, s, True))
        hist = mode in (MODE_WARMUP, MODE_CALIB, MODE_MODEL) and not (self.lanes > 1 and mode == MODE_MODEL)
        self.pending.append((task, v, key, mode, warm, int(cost(v)), hist))
        return v, mode, w

    def sync_all(self):
        self._harvest(lambda p: True)
        self.reset_workers()
