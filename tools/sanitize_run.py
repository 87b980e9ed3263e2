"""Small-shape run of every built-in variant (target for compute-sanitizer memcheck / racecheck /
synccheck): ragged shapes, transB, beta 0 / non-zero, host mode, loopback panels; the sort variants
on ragged n with FP32 keys (incl. multi-tile radix sorts)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import gen  # noqa: E402
from gen.device import device_matrix  # noqa: E402
from paper_2311_03543_b200 import compar as cm  # noqa: E402

only = sys.argv[1:]  # optional variant names
ctx = cm.Compar()
names = [v for v, _ in ctx.variants()]
for name in names:
    if only and name not in only:
        continue
    if name.startswith("sort_"):
        for n in ([2, 1000, 16384] if name == "sort_bitonic" else [2, 1000, 16384, 70001, (1 << 24) + 12345]):
            x = torch.randn(n, device="cuda")
            r = ctx.sort(x, variant_hint=names.index(name))
            assert r.status == 0 and bool((x[1:] >= x[:-1]).all()), (name, n)
        print(f"{name}: ok", flush=True)
        continue
    bf = "bf16" in name
    dt = "bf16" if bf else "f32"
    compute = cm.COMPUTE_BF16 if bf else (cm.COMPUTE_TF32 if "tf32" in name else
                                          cm.COMPUTE_F32_SPLIT if name == "tc_f32x3" else cm.COMPUTE_F32_STRICT)
    shapes = [(77, 136, 72, 0, 0.5, 1), (300, 264, 136, 1, 0.0, 3), (129, 520, 264, 0, -1.0, 2)]
    if name.endswith("_sk"):   # the split-K variant needs >= 64 k-blocks
        shapes = [(77, 136, 4160, 0, 0.5, 1), (300, 264, 8200, 1, 0.0, 3), (129, 520, 4160, 0, -1.0, 2)]
    else:                      # more tiles than CTAs / clusters: the counter-fed tiles after the static first
        shapes.append((4096, 2304, 136 if name.endswith("_ck") else 64, 0, 0.5, 1))
    if name.endswith("_2sm"):  # 64 pair tiles of 256 x 256: the single-wave form (C_in staged in TMEM)
        shapes.append((2048, 2048, 136, 0, 0.5, 1))
    if name == "tc_f32x3":     # several accumulation chunks, ragged last chunk, both B layouts
        shapes += [(300, 264, 2100, 1, 0.5, 1), (129, 520, 1030, 0, 0.0, 1)]
    for (m, n, k, tb, beta, panels) in shapes:
        A = device_matrix(gen.TAG_A, m, k, dtype=dt)
        B = device_matrix(gen.TAG_B, k, n, dtype=dt, transposed=bool(tb))
        Cd = device_matrix(gen.TAG_C, m, n)
        d = cm.make_desc(m, n, k, A=A, B=B, C_in=Cd, C_out=Cd, ldb=(k if tb else n), alpha=1.5, beta=beta,
                         in_dtype=cm.BF16 if bf else cm.F32, compute=compute, transB=tb, panels=panels,
                         variant_hint=names.index(name))
        if names.index(name) not in ctx.eligible(d):   # e.g. tc_*_ck: single-wave shapes only
            print(f"{name}: {m}x{n}x{k} not eligible, skipped", flush=True)
            continue
        r = ctx.run(d)
        assert r.status == 0, (name, m, n, k)
    print(f"{name}: ok", flush=True)
torch.cuda.synchronize()
ctx.terminate()

# world mode (loopback, with the NCCL SM reserve): the wide kernel's fused slab-flag launch plus the
# helper launch sharing its tile counter, row-major (3-D slab map) and transposed B
if not only or any(n.endswith("_2sm_w") for n in only):
    os.environ["COMPAR_BCAST_LOOPBACK"] = "2"
    wctx = cm.Compar(bcast_chunks=4, bcast_ctas=8)
    os.environ.pop("COMPAR_BCAST_LOOPBACK")
    wn = [v for v, _ in wctx.variants()]
    for name in ("tc_bf16_2sm_w", "tc_tf32_2sm_w"):
        bf = "bf16" in name
        dt = "bf16" if bf else "f32"
        for (m, n, k, tb) in ((3000, 4096, 136, 0), (2600, 4096, 264, 1)):
            A = device_matrix(gen.TAG_A, m, k, dtype=dt)
            B = device_matrix(gen.TAG_B, k, n, dtype=dt, transposed=bool(tb))
            Cd = device_matrix(gen.TAG_C, m, n)
            d = cm.make_desc(m, n, k, A=A, B=B, C_in=Cd, C_out=Cd, ldb=(k if tb else n), alpha=1.5, beta=0.5,
                             in_dtype=cm.BF16 if bf else cm.F32, compute=cm.COMPUTE_BF16 if bf else cm.COMPUTE_TF32,
                             transB=tb, world=1, variant_hint=wn.index(name))
            for _ in range(2):
                assert wctx.run(d).status == 0, (name, m, n, k)
        print(f"{name} world loopback: ok", flush=True)
    torch.cuda.synchronize()
    wctx.terminate()
