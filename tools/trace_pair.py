"""Phase stamps of the CTA-pair kernel (tc_gemm_2sm_mc) on small grids: where the fixed per-launch
time goes.  Development aid.

  python tools/trace_pair.py build          # (CPU) library with -DCOMPAR_TRACE -> build_trace/
  python tools/trace_pair.py run M N K ...  # (GPU) stamps of CTAs 0 / 1, in SM cycles from entry

Stamps: 0 entry, 1 init done (barriers, TMEM, cluster sync), 2 first TMA issued, 3 first stage
landed (MMA warp), 4 tile 0 committed, 5 epilogue sees the accumulator, 6 tile 0 stored,
7 stores drained, 8 exit sync; 10 / 11 globaltimer at entry / exit.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
TRACE_DIR = os.path.join(ROOT, "build_trace")

if __name__ == "__main__" and sys.argv[1] == "build":
    # python tools/trace_pair.py build [DIR -DFLAG ...]: extra experiment flags into another dir
    from paper_2311_03543_b200 import build as b
    if len(sys.argv) > 2:
        TRACE_DIR = os.path.join(ROOT, sys.argv[2])
    b.ARCH = b.ARCH + ["-DCOMPAR_TRACE"] + sys.argv[3:]
    b.BUILD = os.path.join(TRACE_DIR, "obj")
    b.LIB = os.path.join(TRACE_DIR, "libcompar.so")
    print(b.build_compar(force=True))
    sys.exit(0)

os.environ["COMPAR_LIB"] = os.environ.get("COMPAR_LIB") or os.path.join(TRACE_DIR, "libcompar.so")
import ctypes  # noqa: E402

import torch  # noqa: E402

import gen  # noqa: E402
from gen.device import device_matrix  # noqa: E402
from paper_2311_03543_b200 import compar as cm  # noqa: E402

lib = ctypes.CDLL(os.environ["COMPAR_LIB"])
ctx = cm.Compar()
names = [v for v, _ in ctx.variants()]
args = [int(x) for x in sys.argv[2:]] or [256, 128, 64]
one_sm = sys.argv[1] in ("run1", "run2")   # run2: the cluster split-K kernel (tc_gemm_ck.cu; stamps
                                           # 1 init, 2 first stage, 3 accumulator complete, 4 after
                                           # cluster barrier 1, 5 partials sent, 6 after barrier 2,
                                           # 7 reduced + stored, 8 exit)   # the 1-SM kernel (tc_gemm.cu; stamps of CTA 0: 0 entry, 1 init,
                                  # 2 first TMA, 3 / 4 first / last stage landed, 5 epilogue sees the
                                  # accumulator, 6 tile stored, 8 exit; 10 / 11 globaltimer)
for i in range(0, len(args), 3):
    m, n, k = args[i:i + 3]
    if one_sm:
        for beta in (0.5, 0.0):
            A = device_matrix(gen.TAG_A, m, k, dtype="bf16")
            B = device_matrix(gen.TAG_B, k, n, dtype="bf16")
            C = device_matrix(gen.TAG_C, m, n)
            d = cm.make_desc(m, n, k, A=A, B=B, C_in=C, C_out=C, alpha=1.5, beta=beta, in_dtype=cm.BF16,
                             compute=cm.COMPUTE_BF16,
                             variant_hint=names.index("tc_bf16_ck" if sys.argv[1] == "run2" else "tc_bf16"))
            for _ in range(5):
                rep = ctx.run(d)
            buf = (ctypes.c_ulonglong * 16)()
            assert (lib.compar_trace2_read if sys.argv[1] == "run2" else lib.compar_trace1_read)(buf) == 0
            t = list(buf)
            st = " ".join(f"{j}:{t[j] - t[0]:6d}" for j in ((1, 2, 3, 4, 5, 6, 7, 8) if sys.argv[1] == "run2"
                                                                 else (1, 2, 3, 4, 5, 6, 8)))
            print(f"1sm {m}x{n}x{k} beta={beta}: {st} | wall {(t[11] - t[10]) / 1e3:.2f} us | event {rep.ns / 1e3:.2f} us",
                  flush=True)
            if sys.argv[1] == "run1":   # entry / exit spread over the CTAs (globaltimer, ns)
                cb = (ctypes.c_ulonglong * 320)()
                assert lib.compar_trace1_cta_read(cb) == 0
                ent = [cb[2 * i] for i in range(160) if cb[2 * i] and cb[2 * i + 1] >= cb[2 * i]]
                ext = [cb[2 * i + 1] for i in range(160) if cb[2 * i] and cb[2 * i + 1] >= cb[2 * i]]
                e0 = min(ent)
                print(f"    ctas {len(ent)}: entry spread {(max(ent) - e0) / 1e3:.2f} us, exit first "
                      f"{(min(ext) - e0) / 1e3:.2f} last {(max(ext) - e0) / 1e3:.2f} us", flush=True)
        continue
    for beta in (0.5, 0.0):
        A = device_matrix(gen.TAG_A, m, k, dtype="bf16")
        B = device_matrix(gen.TAG_B, k, n, dtype="bf16")
        C = device_matrix(gen.TAG_C, m, n)
        d = cm.make_desc(m, n, k, A=A, B=B, C_in=C, C_out=C, alpha=1.5, beta=beta, in_dtype=cm.BF16,
                         compute=cm.COMPUTE_BF16, variant_hint=names.index("tc_bf16_2sm"))
        for _ in range(5):
            rep = ctx.run(d)
        buf = (ctypes.c_ulonglong * 32)()
        assert lib.compar_trace_read(buf) == 0
        for cta in (0, 1):
            t = list(buf[cta * 16:(cta + 1) * 16])
            st = " ".join(f"{j}:{t[j] - t[0]:6d}" for j in list(range(10)) + [12, 13, 14, 15])
            print(f"{m}x{n}x{k} beta={beta} cta{cta}: {st} | wall {(t[11] - t[10]) / 1e3:.2f} us | event {rep.ns / 1e3:.2f} us",
                  flush=True)
        cb = (ctypes.c_ulonglong * 320)()
        assert lib.compar_trace_cta_read(cb) == 0
        ent = [cb[2 * i] for i in range(160) if cb[2 * i] and cb[2 * i + 1] >= cb[2 * i]]
        ext = [cb[2 * i + 1] for i in range(160) if cb[2 * i] and cb[2 * i + 1] >= cb[2 * i]]
        e0 = min(ent)
        print(f"    ctas {len(ent)}: entry spread {(max(ent) - e0) / 1e3:.2f} us, exit first "
              f"{(min(ext) - e0) / 1e3:.2f} last {(max(ext) - e0) / 1e3:.2f} us", flush=True)
ctx.terminate()
