"""Development diagnostic: sampled-entry errors of the tc variants at large shapes."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
from gen.device import device_matrix  # noqa: E402
from oracle import gemm as og  # noqa: E402
from paper_2311_03543_b200 import compar as cm  # noqa: E402


def check(ctx, name, m, n, k, beta=0.5):
    names = [v for v, _ in ctx.variants()]
    bf = name == "tc_bf16"
    dt = "bf16" if bf else "f32"
    A = device_matrix(gen.TAG_A, m, k, dtype=dt)
    B = device_matrix(gen.TAG_B, k, n, dtype=dt)
    Cd = device_matrix(gen.TAG_C, m, n)
    d = cm.make_desc(m, n, k, A=A, B=B, C_in=Cd, C_out=Cd, alpha=1.5, beta=beta,
                     in_dtype=cm.BF16 if bf else cm.F32,
                     compute=cm.COMPUTE_BF16 if bf else cm.COMPUTE_TF32, variant_hint=names.index(name),
                     stream=torch.cuda.current_stream().cuda_stream)
    ctx.run(d)
    torch.cuda.synchronize()
    rows = np.unique(np.concatenate([np.arange(0, m, max(1, m // 24)), [m - 1, 127, 128]]))
    cols = np.unique(np.concatenate([np.arange(0, n, max(1, n // 24)), [n - 1, 255, min(256, n - 1)]]))
    got = Cd[torch.as_tensor(rows, device="cuda")][:, torch.as_tensor(cols, device="cuda")].double().cpu().numpy()
    ref = og.gemm(gen.matrix_rows(gen.TAG_A, rows, k, dtype=dt), gen.matrix_cols(gen.TAG_B, k, cols, dtype=dt),
                  gen.matrix_entries(gen.TAG_C, rows, cols), alpha=1.5, beta=beta, dtype=dt)
    err = np.abs(got - ref) / (np.abs(ref).mean() + 1e-30)
    bad = err > 0.05
    print(f"{name} {m}x{n}x{k}: rel_fro={og.rel_fro(got, ref):.3e}  bad={bad.sum()}/{bad.size}", flush=True)
    if bad.any():
        br, bc = np.nonzero(bad)
        print("   bad rows:", sorted(set(rows[br].tolist()))[:20], flush=True)
        print("   bad cols:", sorted(set(cols[bc].tolist()))[:20], flush=True)
    del A, B, Cd
    torch.cuda.empty_cache()


if __name__ == "__main__":
    ctx = cm.Compar()
    shapes = [("tc_bf16", 8192, 8192, 8192), ("tc_bf16", 16384, 16384, 16384), ("tc_bf16", 32768, 4096, 4096),
              ("tc_bf16", 4096, 32768, 4096), ("tc_bf16", 4096, 4096, 32768), ("tc_bf16", 32768, 32768, 4096),
              ("tc_bf16", 32768, 32768, 32768), ("tc_tf32", 1024, 1024, 1024), ("tc_tf32", 8192, 8192, 8192)]
    for s in shapes:
        try:
            check(ctx, *s)
        except Exception as e:  # noqa: BLE001
            print(s, "FAILED", e, flush=True)
    ctx.terminate()
