"""Thin ctypes binding of include/compar.h (argument marshalling only).

Every step of the hot path — selection, partitioning, broadcast, kernels, timing, history —
runs inside libcompar.so; this module only converts Python/torch arguments into the C
structs and raises on non-OK statuses.  There is no fallback: if the native library is
missing or fails to load, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("COMPAR_LIB", os.path.join(_HERE, "libcompar.so"))

# ---- enums (values restate include/compar.h)
OK, E_INVALID, E_STATE, E_DUPLICATE, E_NO_VARIANT, E_CUDA, E_NCCL, E_TASK_FAILED, E_UNKNOWN_TASK, E_IO, \
    E_FORMAT, E_OOM = range(12)
STATUS_NAMES = ["OK", "E_INVALID", "E_STATE", "E_DUPLICATE", "E_NO_VARIANT", "E_CUDA", "E_NCCL", "E_TASK_FAILED",
                "E_UNKNOWN_TASK", "E_IO", "E_FORMAT", "E_OOM"]
F32, BF16 = 0, 1
COMPUTE_F32_STRICT, COMPUTE_TF32, COMPUTE_BF16, COMPUTE_F32_SPLIT = 0, 1, 2, 3
TGT_SIMT_F32, TGT_TMA_F32, TGT_TC_TF32, TGT_TC_BF16, TGT_USER, TGT_TC2_TF32, TGT_TC2_BF16, TGT_TCW_TF32, TGT_TCW_BF16 = \
    0, 1, 2, 3, 4, 5, 6, 7, 8
TGT_SIMT_BF16 = 9
TGT_TCS_TF32, TGT_TCS_BF16 = 10, 11
TGT_TCK_TF32, TGT_TCK_BF16 = 12, 13
TGT_TCX_F32 = 14
TGT_SORT_RADIX, TGT_SORT_BITONIC = 20, 21
KEY_U32, KEY_I32, KEY_F32 = 0, 1, 2
# built-in targets by precision class (the §8(b) eligibility table; include/compar.h)
TARGETS_STRICT = (TGT_SIMT_F32, TGT_TMA_F32)
TARGETS_TF32 = TARGETS_STRICT + (TGT_TC_TF32, TGT_TC2_TF32, TGT_TCW_TF32, TGT_TCS_TF32, TGT_TCK_TF32)
TARGETS_BF16 = (TGT_TC_BF16, TGT_TC2_BF16, TGT_TCW_BF16, TGT_SIMT_BF16, TGT_TCS_BF16, TGT_TCK_BF16)
TARGETS_F32_SPLIT = TARGETS_STRICT + (TGT_TCX_F32,)
MODE_WARMUP, MODE_CALIB, MODE_MODEL, MODE_EAGER, MODE_HINT, MODE_NOOP, MODE_PREDICT = 0, 1, 2, 3, 4, 5, 6
SCHED_HISTORY, SCHED_EAGER, SCHED_PREDICT = 0, 1, 2
CALIB_INTERLEAVED, CALIB_BLOCKED = 0, 1
WORLD_LOCAL, WORLD_PANELS, WORLD_TASKS = 0, 1, 2
MEM_DEVICE, MEM_HOST = 0, 1
TASK_ALL = (1 << 64) - 1
MAX_PANELS = 8
UNIQUE_ID_BYTES = 128
CE_BLOB_BYTES = 256


class Config(C.Structure):
    _fields_ = [("ngpu", C.c_int), ("device", C.c_int), ("sched", C.c_int), ("calib_k", C.c_int),
                ("calib_warmup", C.c_int), ("perf_model_path", C.c_char_p), ("bcast_chunks", C.c_int),
                ("builtins", C.c_int), ("virtual_clock", C.c_int), ("variant_mask", C.c_int64),
                ("calib_order", C.c_int), ("lanes", C.c_int), ("calib_prune", C.c_int), ("bcast_ctas", C.c_int),
                ("sync_timeout_ms", C.c_int)]


class GemmDesc(C.Structure):
    _fields_ = [("m", C.c_int64), ("n", C.c_int64), ("k", C.c_int64), ("alpha", C.c_float), ("beta", C.c_float),
                ("in_dtype", C.c_int), ("compute", C.c_int), ("transB", C.c_int),
                ("A", C.c_void_p), ("lda", C.c_int64), ("B", C.c_void_p), ("ldb", C.c_int64),
                ("C_in", C.c_void_p), ("ldc_in", C.c_int64), ("C_out", C.c_void_p), ("ldc_out", C.c_int64),
                ("mem", C.c_int), ("stream", C.c_void_p), ("panels", C.c_int), ("world", C.c_int),
                ("B_replica", C.c_void_p), ("variant_hint", C.c_int), ("handles", C.c_uint64 * 4)]


class SortDesc(C.Structure):
    _fields_ = [("n", C.c_int64), ("key_type", C.c_int), ("keys", C.c_void_p), ("stream", C.c_void_p),
                ("variant_hint", C.c_int)]


class Panel(C.Structure):
    _fields_ = [("index", C.c_int), ("row0", C.c_int64), ("rows", C.c_int64), ("A", C.c_void_p),
                ("B", C.c_void_p), ("C_in", C.c_void_p), ("C_out", C.c_void_p)]


class Report(C.Structure):
    _fields_ = [("task", C.c_uint64), ("variant", C.c_int), ("mode", C.c_int), ("warmup", C.c_int),
                ("status", C.c_int), ("npanels", C.c_int), ("ns", C.c_int64),
                ("panel_ns", C.c_int64 * MAX_PANELS), ("bcast_ns", C.c_int64), ("total_ns", C.c_int64),
                ("batch", C.c_int), ("rank", C.c_int), ("lane", C.c_int)]


class Record(C.Structure):
    _fields_ = [("seen", C.c_int64), ("count", C.c_int64), ("min_ns", C.c_int64), ("sum_ns", C.c_int64),
                ("mean_ns", C.c_double)]


class Stats(C.Structure):
    _fields_ = [("submits", C.c_int64), ("launches", C.c_int64), ("harvested", C.c_int64), ("failed", C.c_int64),
                ("bytes_h2d", C.c_int64), ("bytes_d2h", C.c_int64)]


GEMM_FN = C.CFUNCTYPE(C.c_int, C.POINTER(GemmDesc), C.POINTER(Panel), C.c_void_p, C.c_void_p,
                      C.POINTER(C.c_int64))
SORT_FN = C.CFUNCTYPE(C.c_int, C.POINTER(SortDesc), C.c_void_p, C.c_void_p, C.POINTER(C.c_int64))
REDUCE_FN = C.CFUNCTYPE(None, C.POINTER(C.c_int64), C.c_void_p)
GENERIC_FN = C.CFUNCTYPE(C.c_int, C.POINTER(C.c_void_p), C.POINTER(C.c_int64), C.c_int, C.c_void_p)


class GenericDesc(C.Structure):
    _fields_ = [("iface", C.c_char_p), ("nargs", C.c_int), ("args", C.POINTER(C.c_void_p)), ("nsizes", C.c_int),
                ("sizes", C.POINTER(C.c_int64)), ("stream", C.c_void_p), ("variant_hint", C.c_int)]
REDUCE_N_FN = C.CFUNCTYPE(None, C.POINTER(C.c_int64), C.c_int, C.c_void_p)

EXPORTS = ["compar_config_default", "compar_init", "compar_terminate", "compar_register_variant",
           "compar_variant_count", "compar_variant_info", "compar_gemm_submit", "compar_sync", "compar_select",
           "compar_register_sort_variant", "compar_sort_submit",
           "compar_register_generic_variant", "compar_generic_submit", "compar_current_stream",
           "compar_perf_save", "compar_perf_load", "compar_history_get", "compar_partition_rows",
           "compar_comm_unique_id", "compar_comm_init", "compar_world_init", "compar_ce_export", "compar_ce_import",
           "compar_set_reduce_hook", "compar_set_reduce_n_hook",
           "compar_stats_get",
           "compar_last_error", "compar_debug_spin"]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libcompar.so not built at {LIB_PATH} (run python -m paper_2311_03543_b200.build)")
    lib = C.CDLL(LIB_PATH)
    vp, i, i64, st = C.c_void_p, C.c_int, C.c_int64, C.c_int
    sig = {
        "compar_config_default": (None, [C.POINTER(Config)]),
        "compar_init": (st, [C.POINTER(Config), C.POINTER(vp)]),
        "compar_terminate": (st, [vp]),
        "compar_register_variant": (st, [vp, C.c_char_p, C.c_char_p, i, GEMM_FN, vp, C.POINTER(i)]),
        "compar_variant_count": (st, [vp, C.POINTER(i)]),
        "compar_variant_info": (st, [vp, i, C.c_char_p, i, C.POINTER(i)]),
        "compar_gemm_submit": (st, [vp, C.POINTER(GemmDesc), C.POINTER(C.c_uint64)]),
        "compar_register_sort_variant": (st, [vp, C.c_char_p, i, SORT_FN, vp, C.POINTER(i)]),
        "compar_sort_submit": (st, [vp, C.POINTER(SortDesc), C.POINTER(C.c_uint64)]),
        "compar_register_generic_variant": (st, [vp, C.c_char_p, C.c_char_p, GENERIC_FN, vp, C.POINTER(i)]),
        "compar_generic_submit": (st, [vp, C.POINTER(GenericDesc), C.POINTER(C.c_uint64)]),
        "compar_current_stream": (vp, []),
        "compar_sync": (st, [vp, C.c_uint64, C.POINTER(Report)]),
        "compar_select": (st, [vp, C.POINTER(GemmDesc), C.POINTER(i), C.POINTER(i)]),
        "compar_perf_save": (st, [vp, C.c_char_p]),
        "compar_perf_load": (st, [vp, C.c_char_p]),
        "compar_history_get": (st, [vp, i, C.POINTER(GemmDesc), C.POINTER(Record)]),
        "compar_partition_rows": (st, [i64, i, C.POINTER(i64)]),
        "compar_comm_unique_id": (st, [vp, i]),
        "compar_comm_init": (st, [vp, i, i, vp, i]),
        "compar_world_init": (st, [vp, i, i]),
        "compar_ce_export": (st, [vp, i, i, C.c_uint64, vp, i]),
        "compar_ce_import": (st, [vp, vp, i]),
        "compar_set_reduce_hook": (st, [vp, REDUCE_FN, vp]),
        "compar_set_reduce_n_hook": (st, [vp, REDUCE_N_FN, vp]),
        "compar_stats_get": (st, [vp, C.POINTER(Stats)]),
        "compar_last_error": (C.c_char_p, [vp]),
        "compar_debug_spin": (st, [vp, i64]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype, fn.argtypes = res, args
    return lib


lib = _load()


class ComparError(RuntimeError):
    def __init__(self, status, msg):
        self.status = status
        super().__init__(f"{STATUS_NAMES[status] if 0 <= status < len(STATUS_NAMES) else status}: {msg}")


def _check(status, ctx=None):
    if status != OK:
        msg = lib.compar_last_error(ctx)
        raise ComparError(status, msg.decode() if msg else "")
    return status


def current_stream() -> int:
    """compar_current_stream(): the running generic variant's stream (inside a variant call)."""
    return lib.compar_current_stream() or 0


def partition_rows(m: int, p: int) -> list[int]:
    out = (C.c_int64 * (p + 1))()
    _check(lib.compar_partition_rows(m, p, out))
    return list(out)


def comm_unique_id() -> bytes:
    buf = C.create_string_buffer(UNIQUE_ID_BYTES)
    _check(lib.compar_comm_unique_id(buf, UNIQUE_ID_BYTES))
    return buf.raw


def debug_spin(stream, ns: int) -> None:
    _check(lib.compar_debug_spin(stream, int(ns)))


def _ptr(x):
    """Device/host address of a torch tensor, int address, or None."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    return x.data_ptr()


def make_sort_desc(keys, n=None, key_type=None, stream=None, variant_hint=-1) -> SortDesc:
    d = SortDesc()
    if n is None:
        n = keys.numel()
    if key_type is None:
        import torch
        key_type = {torch.float32: KEY_F32, torch.int32: KEY_I32}.get(keys.dtype, KEY_U32)
    d.n, d.key_type, d.keys, d.stream, d.variant_hint = int(n), int(key_type), _ptr(keys), stream, int(variant_hint)
    return d


def make_desc(m, n, k, *, A=None, B=None, C_in=None, C_out=None, lda=None, ldb=None, ldc_in=None, ldc_out=None,
              alpha=1.0, beta=0.0, in_dtype=F32, compute=COMPUTE_F32_STRICT, transB=0, mem=MEM_DEVICE, stream=None,
              panels=0, world=0, B_replica=None, variant_hint=-1, handles=None) -> GemmDesc:
    d = GemmDesc()
    d.m, d.n, d.k = int(m), int(n), int(k)
    d.alpha, d.beta = float(alpha), float(beta)
    d.in_dtype, d.compute, d.transB = int(in_dtype), int(compute), int(transB)
    d.A, d.B, d.C_in, d.C_out = _ptr(A), _ptr(B), _ptr(C_in), _ptr(C_out)
    d.lda = int(lda if lda is not None else (A.stride(0) if hasattr(A, "stride") else k))
    d.ldb = int(ldb if ldb is not None else (B.stride(0) if hasattr(B, "stride") else (k if transB else n)))
    d.ldc_in = int(ldc_in if ldc_in is not None else (C_in.stride(0) if hasattr(C_in, "stride") else n))
    d.ldc_out = int(ldc_out if ldc_out is not None else (C_out.stride(0) if hasattr(C_out, "stride") else n))
    d.mem = int(mem)
    d.stream = stream
    d.panels, d.world = int(panels), int(world)
    d.B_replica = _ptr(B_replica)
    d.variant_hint = int(variant_hint)
    if handles is not None:          # (A, B, C_in, C_out) data-handle ids, 0 = byte range
        for i, h in enumerate(handles):
            d.handles[i] = int(h)
    return d


class Compar:
    """One runtime context (compar_init ... compar_terminate)."""

    def __init__(self, ngpu=-1, device=-1, sched=-1, calib_k=-1, calib_warmup=-1, perf_model_path=None,
                 bcast_chunks=-1, builtins=-1, virtual_clock=0, variant_mask=-1, calib_order=-1, lanes=-1,
                 calib_prune=-1, bcast_ctas=-1, sync_timeout_ms=-1):
        cfg = Config()
        lib.compar_config_default(C.byref(cfg))
        cfg.ngpu, cfg.device, cfg.sched = ngpu, device, sched
        cfg.calib_k, cfg.calib_warmup = calib_k, calib_warmup
        self._path = perf_model_path.encode() if perf_model_path else None
        cfg.perf_model_path = self._path
        cfg.bcast_chunks, cfg.builtins, cfg.virtual_clock = bcast_chunks, builtins, virtual_clock
        cfg.variant_mask = variant_mask
        cfg.calib_order = calib_order
        cfg.lanes = lanes
        cfg.calib_prune, cfg.bcast_ctas, cfg.sync_timeout_ms = calib_prune, bcast_ctas, sync_timeout_ms
        self.ctx = C.c_void_p()
        self._callbacks = []     # keep ctypes thunks alive
        _check(lib.compar_init(C.byref(cfg), C.byref(self.ctx)))

    # lifecycle
    def terminate(self):
        if self.ctx:
            ctx, self.ctx = self.ctx, C.c_void_p()
            _check(lib.compar_terminate(ctx))

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.terminate()

    # variants
    def register_variant(self, name, target=TGT_USER, fn=None, iface="gemm") -> int:
        out = C.c_int()
        cfn = GEMM_FN(fn) if fn is not None else GEMM_FN()
        self._callbacks.append(cfn)
        _check(lib.compar_register_variant(self.ctx, iface.encode() if iface is not None else None,
                                           name.encode() if name is not None else None, target, cfn, None,
                                           C.byref(out)), self.ctx)
        return out.value

    def register_sort_variant(self, name, target=TGT_USER, fn=None) -> int:
        out = C.c_int()
        cfn = SORT_FN(fn) if fn is not None else SORT_FN()
        self._callbacks.append(cfn)
        _check(lib.compar_register_sort_variant(self.ctx, name.encode() if name is not None else None, target, cfn,
                                                None, C.byref(out)), self.ctx)
        return out.value

    def register_generic_variant(self, iface: str, name: str, fn) -> int:
        """A variant of a user interface (what the #pragma compar pre-compiler generates):
        fn(args, sizes, nsizes, user) enqueues GPU work on current_stream()."""
        cfn = GENERIC_FN(fn)
        self._callbacks.append(cfn)
        out = C.c_int()
        _check(lib.compar_register_generic_variant(self.ctx, iface.encode(), name.encode(), cfn, None, C.byref(out)),
               self.ctx)
        return out.value

    def generic_submit(self, iface: str, args_ptrs, sizes, stream=None, variant_hint=-1) -> int:
        arr = (C.c_void_p * max(1, len(args_ptrs)))(*args_ptrs)
        sz = (C.c_int64 * max(1, len(sizes)))(*[int(x) for x in sizes])
        d = GenericDesc(iface.encode(), len(args_ptrs), arr, len(sizes), sz, stream, variant_hint)
        t = C.c_uint64()
        _check(lib.compar_generic_submit(self.ctx, C.byref(d), C.byref(t)), self.ctx)
        return t.value

    def variants(self) -> list[tuple[str, int]]:
        n = C.c_int()
        _check(lib.compar_variant_count(self.ctx, C.byref(n)), self.ctx)
        out = []
        for v in range(n.value):
            buf, tgt = C.create_string_buffer(64), C.c_int()
            _check(lib.compar_variant_info(self.ctx, v, buf, 64, C.byref(tgt)), self.ctx)
            out.append((buf.value.decode(), tgt.value))
        return out

    # tasks
    def submit(self, desc: GemmDesc) -> int:
        t = C.c_uint64()
        _check(lib.compar_gemm_submit(self.ctx, C.byref(desc), C.byref(t)), self.ctx)
        return t.value

    def sync(self, task=TASK_ALL) -> Report:
        r = Report()
        _check(lib.compar_sync(self.ctx, task, C.byref(r)), self.ctx)
        return r

    def sync_status(self, task=TASK_ALL):
        r = Report()
        s = lib.compar_sync(self.ctx, task, C.byref(r))
        return s, r

    def run(self, desc: GemmDesc) -> Report:
        return self.sync(self.submit(desc))

    def sort_submit(self, desc: "SortDesc") -> int:
        t = C.c_uint64()
        _check(lib.compar_sort_submit(self.ctx, C.byref(desc), C.byref(t)), self.ctx)
        return t.value

    def sort(self, keys, n=None, key_type=None, stream=None, variant_hint=-1) -> Report:
        """The sort interface: sort `keys` (a CUDA tensor / device address) in place."""
        return self.sync(self.sort_submit(make_sort_desc(keys, n=n, key_type=key_type, stream=stream,
                                                         variant_hint=variant_hint)))

    def select(self, desc: GemmDesc) -> tuple[int, int]:
        v, m = C.c_int(), C.c_int()
        _check(lib.compar_select(self.ctx, C.byref(desc), C.byref(v), C.byref(m)), self.ctx)
        return v.value, m.value

    def eligible(self, desc: GemmDesc) -> list[int]:
        """Registry indices the selector may pick for this task (§8(c) step 1: precision class, TMA /
        split-K constraints, mask), found by querying compar_select with each variant as a hint."""
        hint = desc.variant_hint
        out = []
        try:
            for v in range(len(self.variants())):
                desc.variant_hint = v
                try:
                    self.select(desc)
                    out.append(v)
                except ComparError:
                    pass
        finally:
            desc.variant_hint = hint
        return out

    # perf model
    def perf_save(self, path):
        _check(lib.compar_perf_save(self.ctx, str(path).encode()), self.ctx)

    def perf_load(self, path):
        _check(lib.compar_perf_load(self.ctx, str(path).encode()), self.ctx)

    def history(self, variant: int, desc: GemmDesc) -> Record:
        r = Record()
        _check(lib.compar_history_get(self.ctx, variant, C.byref(desc), C.byref(r)), self.ctx)
        return r

    # multi-GPU
    def comm_init(self, nranks: int, rank: int, uid: bytes):
        buf = C.create_string_buffer(uid, UNIQUE_ID_BYTES)
        _check(lib.compar_comm_init(self.ctx, nranks, rank, buf, UNIQUE_ID_BYTES), self.ctx)

    def world_init(self, nranks: int, rank: int):
        """SPMD world without NCCL (exchanges through the reduce hooks): compar_world_init."""
        _check(lib.compar_world_init(self.ctx, nranks, rank), self.ctx)

    def ce_init(self, nranks: int, rank: int, max_b_bytes: int, allgather):
        """Copy-engine chain broadcast for world mode (compar_ce_export / _import).  `allgather(b)`
        returns the list of every rank's bytes `b`, rank-major (e.g. torch.distributed
        all_gather_object)."""
        blob = C.create_string_buffer(CE_BLOB_BYTES)
        _check(lib.compar_ce_export(self.ctx, nranks, rank, max_b_bytes, blob, CE_BLOB_BYTES), self.ctx)
        blobs = allgather(bytes(blob.raw))
        allb = C.create_string_buffer(b"".join(blobs), nranks * CE_BLOB_BYTES)
        _check(lib.compar_ce_import(self.ctx, allb, nranks * CE_BLOB_BYTES), self.ctx)

    def set_reduce_hook(self, fn):
        cfn = REDUCE_FN(fn) if fn is not None else REDUCE_FN()
        self._callbacks.append(cfn)
        _check(lib.compar_set_reduce_hook(self.ctx, cfn, None), self.ctx)

    def set_reduce_n_hook(self, fn):
        """fn(buf: POINTER(c_int64), n: int, user) -> None: in-place element-wise max over ranks."""
        cfn = REDUCE_N_FN(fn) if fn is not None else REDUCE_N_FN()
        self._callbacks.append(cfn)
        _check(lib.compar_set_reduce_n_hook(self.ctx, cfn, None), self.ctx)

    def stats(self) -> Stats:
        s = Stats()
        _check(lib.compar_stats_get(self.ctx, C.byref(s)), self.ctx)
        return s
