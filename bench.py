"""bench.py — the measured contract (one JSON line from rank 0).

Workload (BASELINE.json configs[3], "GEMM 32768x32768x32768 row-panel partitioned across
2/4/8 B200 with NCCL broadcast of B"; the metric is quoted at 1/2/4/8 GPUs, and the problem
fits one B200): C = 1.5 * A @ B + 0.5 * C, A/B BF16, C FP32, M = N = K = 32768, A and C
split into 128-aligned row panels over the N ranks, B broadcast from rank 0 with NCCL.
One STEP = one pass of the whole hot path through the C ABI: compar_gemm_submit (validate,
key, select, partition, broadcast, tcgen05 kernel, events) + compar_sync (harvest, history).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--size S]

--gpus N > 1 without torchrun re-executes itself under torch.distributed.run with N ranks; under
torchrun, WORLD_SIZE must equal N.

value = total FLOPs of all ranks / max-over-ranks device time (CUDA events on the launch
stream); inputs (2 GiB + 2 GiB + 4 GiB) are larger than L2, so no flush is needed.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GEMM TFLOP/s at 1/2/4/8 B200 (% of peak); selector regret vs best variant"
ALPHA, BETA = 1.5, 0.5
BAD_REASONS = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown")


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="native", choices=["native", "reference"])
    p.add_argument("--size", type=int, default=32768)
    p.add_argument("--e2e-steps", type=int, default=3)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-targets", action="store_true", help="skip the config-3 / 5a north-star block")
    p.add_argument("--no-yardstick", action="store_true", help="skip the same-operation cuBLAS comparison")
    p.add_argument("--bcast", default="nccl", choices=["nccl", "ce"],
                   help="N > 1: broadcast of B by NCCL (default) or by the copy-engine chain (compar_ce_*)")
    p.add_argument("--variant", default=None, help="testing: force this variant (no selector)")
    p.add_argument("--dump-c", default=None, help="testing: after the run, recompute one step from fresh inputs "
                                                 "and save this rank's C panel to DIR/c_r<rank>.npy")
    return p.parse_args()


def free_port() -> int:
    import socket
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def self_launch(args):
    """`python bench.py --gpus N` (N > 1) outside torchrun: re-exec this script as N ranks under
    torch.distributed.run (one process per GPU, rendezvous on 127.0.0.1) and exit with its code,
    so the driver's plain command form measures N GPUs.  NCCL's INIT log lines (communicator
    size per rank) go to stderr."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd, env=env))


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            mp = json.load(f)
        return mp, "measured"
    except (OSError, ValueError):
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "sm_max_mhz": 1965.0}, \
            "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region (B200_PROFILING.md)."""
    FIELDS = ["clocks.sm", "clocks.max.sm", "power.draw", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            t0 = time.time()
            while not self.lines and time.time() - t0 < 3.0:   # sampler live before the timed region
                time.sleep(0.01)
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, smax, reasons, power = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) != len(self.FIELDS):
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
                power.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        loaded = [s for s in sm if smax and s > 0.3 * smax] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w_max": max(power) if power else None}


# ---------------------------------------------------------------------------------------------
def reference_arm(args, rank, world):
    """--impl reference: the FP64 oracle (the reference arm for this tier) on the host cores,
    each step a bounded sample of the same workload (rows x cols sub-block, full K)."""
    if rank != 0:
        return
    import numpy as np

    import gen
    from oracle import gemm as og
    og.set_threads(len(os.sched_getaffinity(0)))   # torchrun exports OMP_NUM_THREADS=1
    M = N = K = args.size
    r = c = 512
    rows = np.linspace(0, M - 1, r).astype(np.int64)
    cols = np.linspace(0, N - 1, c).astype(np.int64)
    Ar = gen.matrix_rows(gen.TAG_A, rows, K, dtype="bf16")
    Bc = gen.matrix_cols(gen.TAG_B, K, cols, dtype="bf16")
    C0 = gen.matrix_entries(gen.TAG_C, rows, cols)
    for _ in range(args.warmup):
        og.gemm(Ar, Bc, C0, alpha=ALPHA, beta=BETA, dtype="bf16")
    t0 = time.perf_counter()
    for _ in range(args.steps):
        og.gemm(Ar, Bc, C0, alpha=ALPHA, beta=BETA, dtype="bf16")
    dt = (time.perf_counter() - t0) / max(args.steps, 1)
    flops = 2.0 * r * c * K
    val = flops / dt / 1e12
    sample = f"{r} rows x {c} cols x full K={K} of the {M}^3 workload per step (FP64 oracle, host cores)"
    out = {"impl": "reference", "metric": METRIC, "value": val, "unit": "TFLOP/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": f"gemm {M}x{N}x{K} bf16 inputs (oracle sample)", "m": M, "n": N, "k": K},
           "cpu_baseline": {"value": val, "unit": "TFLOP/s", "cores": og.threads(), "kind": "oracle",
                            "sample": sample},
           "e2e": {"value": val, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def cpu_baseline(size):
    """The oracle as it stands, timed on the box's host cores on a bounded sample (~10 s)."""
    import numpy as np

    import gen
    from oracle import gemm as og
    og.set_threads(len(os.sched_getaffinity(0)))
    K = size
    r = 256
    for _ in range(3):
        rows = np.linspace(0, size - 1, r).astype(np.int64)
        Ar = gen.matrix_rows(gen.TAG_A, rows, K, dtype="bf16")
        Bc = gen.matrix_cols(gen.TAG_B, K, rows, dtype="bf16")
        C0 = gen.matrix_entries(gen.TAG_C, rows, rows)
        t0 = time.perf_counter()
        og.gemm(Ar, Bc, C0, alpha=ALPHA, beta=BETA, dtype="bf16")
        dt = time.perf_counter() - t0
        if dt > 5.0 or r >= 2048:
            break
        r = min(2048, int(r * max(1.5, (10.0 / max(dt, 1e-3)) ** 0.5)))
    cores = og.threads()
    # the same oracle on ONE thread, on a proportionally smaller sample (~3 s)
    r1 = max(16, int(r / max(cores, 1) ** 0.5))
    rows1 = np.linspace(0, size - 1, r1).astype(np.int64)
    A1 = gen.matrix_rows(gen.TAG_A, rows1, K, dtype="bf16")
    B1 = gen.matrix_cols(gen.TAG_B, K, rows1, dtype="bf16")
    C1 = gen.matrix_entries(gen.TAG_C, rows1, rows1)
    og.set_threads(1)
    t0 = time.perf_counter()
    og.gemm(A1, B1, C1, alpha=ALPHA, beta=BETA, dtype="bf16")
    dt1 = time.perf_counter() - t0
    og.set_threads(cores)
    cpu_model = None
    try:
        with open("/proc/cpuinfo") as f:
            cpu_model = next((ln.split(":", 1)[1].strip() for ln in f if ln.startswith("model name")), None)
    except OSError:
        pass
    return {"value": 2.0 * r * r * K / dt / 1e12, "unit": "TFLOP/s", "cores": cores, "kind": "oracle",
            "sample": f"{r}x{r} sub-block (rows/cols spread over the matrix) x full K={K}, FP64, {dt:.1f} s",
            "value_1_thread": 2.0 * r1 * r1 * K / dt1 / 1e12,
            "sample_1_thread": f"{r1}x{r1} sub-block x full K={K}, FP64, 1 thread, {dt1:.1f} s",
            "cpu_model": cpu_model, "affinity_cores": len(os.sched_getaffinity(0))}


# ---------------------------------------------------------------------------------------------
def pcie_peaks(nbytes=1 << 30, reps=3):
    """Measured host<->device copy peaks on this box (pinned host memory, CUDA events, best of
    `reps`): H2D, D2H, and both directions at once on two streams — the roofline of `e2e`, whose
    timed region moves A, B, C_in up and C_out down."""
    import torch
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    h2 = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn):
        best = None
        for _ in range(reps):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            best = ms if best is None else min(best, ms)
        return best

    h2d = nbytes / timed(lambda: d.copy_(h, non_blocking=True)) / 1e6
    d2h = nbytes / timed(lambda: h.copy_(d, non_blocking=True)) / 1e6

    def both():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)
    bidir = 2 * nbytes / timed(both) / 1e6
    del h, h2, d, d2
    torch.cuda.empty_cache()
    return {"h2d_gbs": h2d, "d2h_gbs": d2h, "bidir_gbs": bidir, "bytes": nbytes,
            "how": "pinned host <-> device copy of 1 GiB, best of 3, CUDA events; bidir = both at once"}


# ---------------------------------------------------------------------------------------------
def fair_medians(ctx, descs, rounds=3, per_round=2, idle_s=0.1):
    """Per-variant time for the regret comparison, robust to the 1 kW power cap: a kernel that
    follows an idle gap or a lower-power kernel runs at boost clocks for a while, so in every round
    each variant gets the same idle gap and one untimed warm-up launch before `per_round` timed
    launches, and the variant order is rotated between rounds.  Returns the median over rounds of
    the per-round mean (ns)."""
    import statistics

    import torch
    vs = list(descs)
    res = {v: [] for v in vs}
    for r in range(rounds):
        order = vs[r % len(vs):] + vs[:r % len(vs)]
        for v in order:
            torch.cuda.synchronize()
            time.sleep(idle_s)
            ctx.run(descs[v])
            res[v].append(sum(ctx.run(descs[v]).ns for _ in range(per_round)) / per_round)
    return {v: statistics.median(x) for v, x in res.items()}


# ---------------------------------------------------------------------------------------------
def cublas_yardstick(ctx, dv, A, B, Cm, M, N, flops_step):
    """cuBLAS on the same operation (C_out = ALPHA*AB + BETA*C_in, FP32 C in and out) at the bench
    shape, interleaved launch by launch with the chosen variant (context, not a bench value)."""
    import torch
    cout = torch.empty((M, N), dtype=torch.float32, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def cublas_once():
        e0.record()
        torch.addmm(Cm, A, B, beta=BETA, alpha=ALPHA, out_dtype=torch.float32, out=cout)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) * 1e6
    cublas_once()
    ctx.run(dv)
    ours_ns, cub_ns = [], []
    for _ in range(3):
        ours_ns.append(ctx.run(dv).ns)
        cub_ns.append(cublas_once())
    yard = {"what": "torch.addmm(C, A, B, beta, alpha, out_dtype=float32): the same operation through cuBLAS",
            "cublas_tflops": flops_step / statistics.median(cub_ns) / 1e3,
            "ours_tflops": flops_step / statistics.median(ours_ns) / 1e3, "launches_each": 3}
    yard["ours_over_cublas"] = yard["ours_tflops"] / yard["cublas_tflops"]
    del cout
    torch.cuda.empty_cache()
    return yard


def alu_peak_tflops(peaks):
    """FP32 FFMA ceiling: SMs x 128 FFMA/clk x 2 FLOP x the max SM clock."""
    import torch
    sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    return sms * 128 * 2 * peaks.get("sm_max_mhz", 1965.0) * 1e6 / 1e12


# (key, m, n, k, storage, compute class) of the BASELINE.json north-star targets timed after the
# headline: config 3 in BF16 (target >= 70 % of the burst BF16 peak), config 5a (HBM-bound), and
# the paper's own arithmetic with FP32 storage ("float arrays", P:202 SGEMM): TF32 tensor
# cores at the headline 32768^3 shape, strict FP32 (FFMA variants only) at 8192^3, and FP32 accuracy
# on tensor cores (class F32_SPLIT, R38: three TF32 products per product) at both.
TARGETS = (("config3_8192cube_bf16", 8192, 8192, 8192, "bf16", "bf16"),
           ("config5a_65536x256x4096_bf16", 65536, 256, 4096, "bf16", "bf16"),
           ("config4_32768cube_tf32_fp32_storage", 32768, 32768, 32768, "f32", "tf32"),
           ("config3_8192cube_f32_strict", 8192, 8192, 8192, "f32", "f32"),
           ("config3_8192cube_f32_split", 8192, 8192, 8192, "f32", "f32x3"),
           ("config4_32768cube_f32_split", 32768, 32768, 32768, "f32", "f32x3"))


def north_star_targets(ctx, cm, peaks, R=10):
    """BASELINE.json north_star targets on this GPU, through the same C ABI (untimed w.r.t. the
    headline).  Each shape: selector trained on the key (calibration), R model-mode runs after an
    idle gap; then regret = chosen / best - 1 over an exhaustive timing of every eligible variant
    of the key's fastest class under fair_medians (the others: their calibration mean).
    Roofline fractions: BF16 against the measured burst BF16 peak, TF32 against half of it (the
    guide's nominal TF32:BF16 ratio), FP32 against the FFMA ALU ceiling, bytes against HBM."""
    import statistics

    import torch

    import gen
    from gen.device import device_matrix
    names = [n for n, _ in ctx.variants()]
    out = {}
    alu = alu_peak_tflops(peaks)
    for key, m, n, k, sdt, cls in TARGETS:
        A = device_matrix(gen.TAG_A, m, k, dtype=sdt)
        B = device_matrix(gen.TAG_B, k, n, dtype=sdt)
        C = device_matrix(gen.TAG_C, m, n)
        compute = {"bf16": cm.COMPUTE_BF16, "tf32": cm.COMPUTE_TF32, "f32": cm.COMPUTE_F32_STRICT,
                   "f32x3": cm.COMPUTE_F32_SPLIT}[cls]
        in_dtype = cm.BF16 if sdt == "bf16" else cm.F32

        def mk(hint=-1):
            return cm.make_desc(m, n, k, A=A, B=B, C_in=C, C_out=C, alpha=ALPHA, beta=BETA, in_dtype=in_dtype,
                                compute=compute, variant_hint=hint)
        d = mk()
        calib = 0
        t_cal = time.perf_counter()
        while ctx.select(d)[1] != cm.MODE_MODEL and calib < 64:
            ctx.run(d)
            calib += 1
        t_cal = time.perf_counter() - t_cal
        torch.cuda.synchronize()
        time.sleep(0.5)                      # same starting power state for every target
        reps = R if m * n * k <= 8192 ** 3 else max(3, R // 2)
        sel = [ctx.run(d) for _ in range(reps)]
        chosen = sel[-1].variant
        E = ctx.eligible(d)
        fast = [v for v in E if names[v].startswith("tc_")] or list(E)
        fm = fair_medians(ctx, {v: mk(v) for v in fast}, rounds=3, per_round=2 if m * n * k > 8192 ** 3 else 3)
        med = {names[v]: fm[v] for v in fast}
        pruned = []
        for v in E:
            if v not in fast:
                h = ctx.history(v, d)
                if h.count:
                    med[names[v]] = h.mean_ns
                else:                      # never launched: pruned by its static lower bound (R32)
                    pruned.append(names[v])
        best = min(med, key=med.get)
        t_sel = statistics.median(r.ns for r in sel)
        flops = 2.0 * m * n * k
        eb = 2 if sdt == "bf16" else 4
        nbytes = eb * (m * k + k * n) + 4 * m * n * 2
        tflops = flops / t_sel / 1e3
        peak = {"bf16": peaks["bf16_tflops"], "tf32": peaks["bf16_tflops"] / 2.0, "f32": alu,
                "f32x3": peaks["bf16_tflops"] / 6.0}[cls]
        out[key] = {"variant": names[chosen], "ms": t_sel / 1e6, "tflops": tflops,
                    "peak_tflops": peak, "frac_of_peak": tflops / peak,
                    "peak_kind": {"bf16": "measured burst BF16 (MEASURED_PEAKS.bf16_tflops)",
                                  "tf32": "half the measured burst BF16 peak (nominal TF32 = BF16 / 2)",
                                  "f32": "FFMA ceiling: SMs x 128 x 2 x sm_max_mhz",
                                  "f32x3": "a third of half the measured burst BF16 peak (three TF32 "
                                           "products per FP32 product)"}[cls],
                    "hbm_gbs": nbytes / t_sel, "frac_of_hbm_peak": nbytes / t_sel / peaks["hbm_gbs"],
                    "best_variant": best, "regret": med[names[chosen]] / med[best] - 1.0,
                    "median_ns_per_variant": med, "pruned_unlaunched": pruned, "calibration_runs": calib,
                    "calibration_s": t_cal}
        if cls == "bf16":
            out[key]["frac_of_bf16_burst_peak"] = tflops / peaks["bf16_tflops"]
        if cls == "tf32":
            out[key]["frac_of_tf32_sustained"] = tflops / (peaks.get("bf16_tflops_sustained", peak * 2) / 2.0)
        if cls in ("f32", "f32x3"):
            out[key]["fp32_alu_peak_tflops"] = alu
            out[key]["over_fp32_alu_peak"] = tflops / alu
        del A, B, C
        torch.cuda.empty_cache()
    out["selector_regret_max"] = max(v["regret"] for v in out.values() if isinstance(v, dict))
    return out


# ---------------------------------------------------------------------------------------------
def main():
    args = parse()
    self_launch(args)
    rank, world, local = dist_env()
    if world != args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU"}), flush=True)
        sys.exit(2)
    if args.impl == "reference":
        reference_arm(args, rank, world)
        return
    import torch
    import torch.distributed as dist

    import gen
    from gen.device import fill
    from paper_2311_03543_b200 import compar as cm

    # COMPAR_BENCH_SHARED_GPU=1 (testing only): every rank on cuda:0 with a gloo process group, so
    # the N > 1 path (with --bcast ce) runs end to end on a one-GPU box; never a performance number
    shared = os.environ.get("COMPAR_BENCH_SHARED_GPU") == "1"
    coll_dev = "cpu" if shared else "cuda"
    if not shared and torch.cuda.device_count() < world:
        print(json.dumps({"error": f"{world} ranks but {torch.cuda.device_count()} visible GPU(s)"}), flush=True)
        sys.exit(2)
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")          # communicator size per rank (INIT lines)
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    torch.cuda.set_device(0 if shared else local)
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    M = N = K = args.size
    offs = cm.partition_rows(M, world)
    r0, r1 = offs[rank], offs[rank + 1]
    mloc = r1 - r0
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream

    ctx = cm.Compar()
    if world > 1:
        if args.bcast == "ce":   # copy-engine chain over CUDA IPC (no NCCL, no SMs; include/compar.h)
            def allgather(b):
                out = [None] * world
                dist.all_gather_object(out, b)
                return out

            def red(p, _user):
                t = torch.tensor([p[0]], dtype=torch.int64, device=coll_dev)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                p[0] = int(t.item())
            ctx.ce_init(world, rank, K * N * 2, allgather)
            ctx.set_reduce_hook(red)
        else:
            uid = [cm.comm_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(uid, src=0)
            ctx.comm_init(world, rank, uid[0])
    # inputs resident in HBM: this rank's A/C panels, B on rank 0 (replica buffer elsewhere)
    A = torch.empty((max(mloc, 1), K), dtype=torch.bfloat16, device="cuda")
    Cm = torch.empty((max(mloc, 1), N), dtype=torch.float32, device="cuda")
    B = torch.empty((K, N), dtype=torch.bfloat16, device="cuda")
    if mloc > 0:
        fill(A.data_ptr(), "bf16", mloc, K, K, gen.TAG_A, row0=r0, stream=sp)
        fill(Cm.data_ptr(), "f32", mloc, N, N, gen.TAG_C, row0=r0, stream=sp)
    if rank == 0:
        fill(B.data_ptr(), "bf16", K, N, N, gen.TAG_B, stream=sp)
    torch.cuda.synchronize()
    hint = [v for v, _ in ctx.variants()].index(args.variant) if args.variant else -1
    desc = cm.make_desc(M, N, K, A=A, B=B if rank == 0 else None, C_in=Cm, C_out=Cm, lda=K, ldb=N, ldc_in=N,
                        ldc_out=N, alpha=ALPHA, beta=BETA, in_dtype=cm.BF16, compute=cm.COMPUTE_BF16, stream=sp,
                        world=1 if world > 1 else 0, B_replica=B if rank != 0 else None, variant_hint=hint)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(n_steps, d):
        reports = []
        barrier()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st0 = ctx.stats()
        ev0.record(stream)
        for _ in range(n_steps):
            reports.append(ctx.run(d))
        ev1.record(stream)
        barrier()
        st1 = ctx.stats()
        ms = ev0.elapsed_time(ev1)
        if world > 1:
            t = torch.tensor([ms], device=coll_dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms, reports, st1.launches - st0.launches

    # Selector training (setup, untimed): run the hot path until the history selector leaves
    # calibration for this key (W warm-up + K timed samples per eligible variant), as a StarPU
    # application does before its measured runs; then the W warm-up steps of the contract.
    calib_runs = 0
    while hint < 0 and ctx.select(desc)[1] != cm.MODE_MODEL and calib_runs < 64:
        ctx.run(desc)
        calib_runs += 1
    for _ in range(args.warmup):
        ctx.run(desc)
    clk = ClockSampler(0 if shared else local)
    clk.start()
    ms, reps, launches = timed(args.steps, desc)
    clocks = clk.stop()
    if any(r in clocks.get("reasons", []) for r in BAD_REASONS):   # rejected: re-measure once
        clk = ClockSampler(0 if shared else local)
        clk.start()
        ms, reps, launches = timed(args.steps, desc)
        clocks = clk.stop()
        clocks["remeasured"] = True

    flops_step = 2.0 * M * N * K
    value = flops_step * args.steps / (ms * 1e-3) / 1e12
    # roofline of the dominant kernel: tcgen05 tc_bf16 panel GEMM, per-launch device time from the
    # task reports (CUDA events on the launch stream, inside the timed region)
    kern_ns = [r.ns for r in reps]
    k_avg = sum(kern_ns) / len(kern_ns)
    if world > 1:
        t = torch.tensor([k_avg], device=coll_dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        k_avg = float(t.item())
    panel_flops = 2.0 * (offs[1] - offs[0]) * N * K
    achieved = panel_flops / (k_avg * 1e-9) / 1e12
    peaks, src = load_peaks()
    peak = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops"))
    variant_names = [v for v, _ in ctx.variants()]
    chosen = variant_names[reps[-1].variant] if reps[-1].variant >= 0 else None
    used = sorted({variant_names[r.variant] for r in reps if r.variant >= 0})
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(prof):     # per-launch DRAM bytes of the timed kernel from the committed ncu capture
        try:
            with open(prof) as f:
                traffic = json.load(f).get(f"{chosen}_{offs[1] - offs[0]}", {}).get("dram_bytes_per_launch")
        except (OSError, ValueError):
            traffic = None
    bcast_ms = sum(r.bcast_ns for r in reps) / len(reps) / 1e6

    # selector regret at the headline key (after the timed region): every eligible tensor-core
    # variant timed 3x, interleaved, through the same call with a variant hint; FFMA variants use
    # their calibration mean (they are ~30x slower here)
    regret = None
    if world == 1:
        vn = [v for v, _ in ctx.variants()]
        elig = ctx.eligible(desc)
        tcv = [v for v in elig if vn[v].startswith("tc_")]
        hinted = {v: cm.make_desc(M, N, K, A=A, B=B, C_in=Cm, C_out=Cm, lda=K, ldb=N, ldc_in=N, ldc_out=N,
                                  alpha=ALPHA, beta=BETA, in_dtype=cm.BF16, compute=cm.COMPUTE_BF16, stream=sp,
                                  variant_hint=v) for v in tcv}
        fm = fair_medians(ctx, hinted, rounds=3, per_round=2)
        med = {vn[v]: fm[v] for v in tcv}
        pruned = []
        for v in elig:
            if v not in tcv:
                h = ctx.history(v, desc)
                if h.count:
                    med[vn[v]] = h.mean_ns
                else:                      # never launched: pruned by its static lower bound (R32)
                    pruned.append(vn[v])
        best = min(med, key=med.get)
        regret = {"chosen": vn[reps[-1].variant], "best": best,
                  "regret": med[vn[reps[-1].variant]] / med[best] - 1.0, "median_ns_per_variant": med,
                  "pruned_unlaunched": pruned}

    # context, not a bench value: cuBLAS on the SAME operation at this shape (torch.addmm with FP32
    # C in and out, out_dtype=float32), interleaved launch by launch with the chosen variant
    yard = None
    if world == 1 and not args.no_yardstick:
        try:
            yard = cublas_yardstick(ctx, hinted[reps[-1].variant] if reps[-1].variant in hinted else desc,
                                    A, B, Cm, M, N, flops_step)
        except Exception as ex:  # noqa: BLE001  (context only: never fail the bench on it)
            yard = {"error": str(ex)[:200]}

    # end to end through the same C ABI call with HOST buffers (pinned), copies in the timed region
    e2e = None
    if args.e2e_steps > 0:
        Ah = A.cpu().pin_memory() if mloc > 0 else torch.empty(0, dtype=torch.bfloat16).pin_memory()
        Ch = Cm.cpu().pin_memory()
        Bh = B.cpu().pin_memory() if rank == 0 else None
        del A
        torch.cuda.empty_cache()
        dh = cm.make_desc(M, N, K, A=Ah, B=Bh, C_in=Ch, C_out=Ch, lda=K, ldb=N, ldc_in=N, ldc_out=N, alpha=ALPHA,
                          beta=BETA, in_dtype=cm.BF16, compute=cm.COMPUTE_BF16, stream=sp, mem=cm.MEM_HOST,
                          world=1 if world > 1 else 0, B_replica=B if rank != 0 else None)
        ctx.run(dh)
        s0 = ctx.stats()
        ems, _, _ = timed(args.e2e_steps, dh)
        s1 = ctx.stats()
        h2d = (s1.bytes_h2d - s0.bytes_h2d) // args.e2e_steps
        d2h = (s1.bytes_d2h - s0.bytes_d2h) // args.e2e_steps
        e2e = {"value": flops_step * args.e2e_steps / (ems * 1e-3) / 1e12, "unit": "TFLOP/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "steps": args.e2e_steps,
               "ms_per_step": ems / args.e2e_steps}
        if world == 1:   # the link's own roofline: the step's bytes at the measured copy peaks
            pk = pcie_peaks()
            floor_ms = max((h2d + d2h) / (pk["bidir_gbs"] * 1e9), h2d / (pk["h2d_gbs"] * 1e9),
                           d2h / (pk["d2h_gbs"] * 1e9)) * 1e3
            e2e["roofline"] = {"bound": "pcie", "peaks": pk,
                               "achieved_gbs": (h2d + d2h) / (e2e["ms_per_step"] * 1e-3) / 1e9,
                               "floor_ms_per_step": floor_ms,
                               "frac": floor_ms / e2e["ms_per_step"]}
        if world > 1:
            t = torch.tensor([h2d, d2h], device=coll_dev, dtype=torch.float64)
            dist.all_reduce(t)
            e2e["h2d_bytes_per_step"], e2e["d2h_bytes_per_step"] = int(t[0].item()), int(t[1].item())

    targets = None
    if world == 1 and not args.no_targets:
        del Cm
        torch.cuda.empty_cache()
        targets = north_star_targets(ctx, cm, load_peaks()[0])

    if args.dump_c:    # testing: one fresh step, this rank's C panel saved (bitwise comparison across N)
        import numpy as np
        Cd = torch.empty((max(mloc, 1), N), dtype=torch.float32, device="cuda")
        Ad = torch.empty((max(mloc, 1), K), dtype=torch.bfloat16, device="cuda")
        if mloc > 0:
            fill(Ad.data_ptr(), "bf16", mloc, K, K, gen.TAG_A, row0=r0, stream=sp)
            fill(Cd.data_ptr(), "f32", mloc, N, N, gen.TAG_C, row0=r0, stream=sp)
        if rank == 0:
            fill(B.data_ptr(), "bf16", K, N, N, gen.TAG_B, stream=sp)
        torch.cuda.synchronize()
        dd = cm.make_desc(M, N, K, A=Ad, B=B if rank == 0 else None, C_in=Cd, C_out=Cd, lda=K, ldb=N, ldc_in=N,
                          ldc_out=N, alpha=ALPHA, beta=BETA, in_dtype=cm.BF16, compute=cm.COMPUTE_BF16, stream=sp,
                          world=1 if world > 1 else 0, B_replica=B if rank != 0 else None,
                          variant_hint=reps[-1].variant)
        ctx.run(dd)
        os.makedirs(args.dump_c, exist_ok=True)
        np.save(os.path.join(args.dump_c, f"c_r{rank}.npy"), Cd[:mloc].cpu().numpy())
        del Cd, Ad

    out = None
    if rank == 0:
        out = {"metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
               "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
               "config": {"workload": f"BASELINE config 4: gemm {M}x{N}x{K}, A/B bf16, C fp32, C=1.5AB+0.5C, "
                                      f"row panels over {world} GPU(s) + "
                                      f"{'copy-engine chain' if args.bcast == 'ce' else 'NCCL'} broadcast of B",
                          "m": M, "n": N, "k": K, "global_batch": None, "seq_len": None,
                          "parallelism": f"rowpanel{world}", "variant": chosen,
                          "bcast": (args.bcast if world > 1 else None),
                          "l2": "inputs larger than L2 (A,B 2 GiB bf16; C 4 GiB fp32): no flush needed"},
               "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                            "frac": achieved / peak, "traffic": traffic,
                            "kernel": "tc_gemm<bf16> (tcgen05/TMEM, persistent, 1 launch per step per GPU)",
                            "peak_source": f"{src} bf16_tflops_sustained (kernel runs back to back)",
                            "frac_of_burst": achieved / peaks.get("bf16_tflops", peak),
                            "avg_launch_ms": k_avg / 1e6},
               "pct_of_peak": value / peak * 100.0,
               "step_kernel_ms": {"mean": k_avg / 1e6, "median": statistics.median(kern_ns) / 1e6,
                                  "min": min(kern_ns) / 1e6, "n": len(kern_ns)},
               "bcast_ms_per_step": bcast_ms,
               "gpu_launches": int(launches),
               "selector": {"calibration_runs_before_timing": calib_runs, "chosen": chosen, "regret": regret,
                            "variants_in_timed_region": used,
                            "eligible": [variant_names[v] for v in ctx.eligible(desc)]},
               "clocks": clocks, "e2e": e2e, "north_star_targets": targets, "cublas_same_op": yard}
        # tensor utilisation from FLOP per SM-cycle at the clock sampled under load (ncu's
        # tensor-pipe-active counter under-reports the CTA-pair kernels): a BF16 tcgen05 M=128 N=256
        # K=16 MMA per SM retires 2*128*256*16 FLOP in 128 cycles = 8192 FLOP / SM-cycle
        sm_mhz = (clocks or {}).get("sm_mhz")
        if sm_mhz:
            sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
            per = achieved * 1e12 / (sms * sm_mhz * 1e6)
            out["roofline"]["per_sm_cycle"] = {"flop_per_sm_cycle": per, "peak_flop_per_sm_cycle": 8192,
                                               "frac": per / 8192, "sms": sms, "sm_mhz": sm_mhz}
    if world > 1:
        dist.barrier()
    ctx.terminate()
    if rank == 0:
        if world == 1 and not args.no_cpu_baseline:
            del B
            out["cpu_baseline"] = cpu_baseline(args.size)
        else:
            out["cpu_baseline"] = None
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
