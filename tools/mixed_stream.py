"""Task-parallel world on one B200: BASELINE config 5b's mixed stream (200 tasks,
shapes drawn with numpy PCG64 seed 7, FP32 under COMPUTE_TF32, beta = 0) submitted as
world = COMPAR_WORLD_TASKS with 1, 2 and 4 lanes, plus a stream of small independent GEMMs where
lane concurrency matters.  Each configuration: one calibration pass, then timed passes (host wall
clock around submit-all + sync-all, GPU idle before and after).
usage: python tools/mixed_stream.py [out.json]
"""
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
from gen.device import device_matrix  # noqa: E402
from paper_2311_03543_b200 import compar as cm  # noqa: E402


def run(stream, probs, lanes, passes=3):
    ctx = cm.Compar(lanes=lanes)
    st = torch.cuda.current_stream().cuda_stream

    def one_pass():
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for s in stream:
            A, B, C = probs[s]
            ctx.submit(cm.make_desc(s[0], s[1], s[2], A=A, B=B, C_in=C, C_out=C, alpha=1.5, beta=0.0,
                                    compute=cm.COMPUTE_TF32, world=cm.WORLD_TASKS, stream=st))
        ctx.sync()
        torch.cuda.synchronize()
        return time.perf_counter() - t0
    cal = one_pass()
    ts = [one_pass() for _ in range(passes)]
    ctx.terminate()
    return {"calibration_pass_s": cal, "pass_s": ts, "median_s": statistics.median(ts)}


def main(out):
    torch.cuda.set_device(0)
    shapes = [(64, 64, 64), (256, 256, 256), (1024, 1024, 1024), (4096, 4096, 4096), (8192, 8192, 8192),
              (65536, 256, 4096), (4096, 4096, 256)]
    rng = np.random.Generator(np.random.PCG64(7))
    stream = [shapes[i] for i in rng.integers(0, len(shapes), 200)]
    probs = {s: (device_matrix(gen.TAG_A, s[0], s[2]), device_matrix(gen.TAG_B, s[2], s[1]),
                 device_matrix(gen.TAG_C, s[0], s[1])) for s in shapes}
    res = {"config5b": {f"lanes{L}": run(stream, probs, L) for L in (1, 2, 4)}}
    del probs
    torch.cuda.empty_cache()
    # small independent GEMMs: 400 tasks over 16 distinct outputs, sizes 128..512
    small = [(128, 128, 128), (256, 256, 256), (384, 384, 384), (512, 512, 512)]
    probs = {}
    stream = []
    for i in range(16):
        s = small[i % 4]
        key = (s[0], s[1], s[2], i)
        probs[key] = (device_matrix(gen.TAG_A, s[0], s[2]), device_matrix(gen.TAG_B, s[2], s[1]),
                      torch.zeros(s[0], s[1], device="cuda"))
    keys = list(probs)
    stream = [keys[i % 16] for i in range(400)]

    def run_small(lanes):
        ctx = cm.Compar(lanes=lanes)
        st = torch.cuda.current_stream().cuda_stream

        def one_pass():
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for key in stream:
                A, B, C = probs[key]
                ctx.submit(cm.make_desc(key[0], key[1], key[2], A=A, B=B, C_in=C, C_out=C, alpha=1.0, beta=0.0,
                                        compute=cm.COMPUTE_TF32, world=cm.WORLD_TASKS, stream=st))
            ctx.sync()
            torch.cuda.synchronize()
            return time.perf_counter() - t0
        one_pass()
        ts = [one_pass() for _ in range(3)]
        ctx.terminate()
        return {"pass_s": ts, "median_s": statistics.median(ts)}
    res["small400"] = {f"lanes{L}": run_small(L) for L in (1, 2, 4)}
    txt = json.dumps(res, indent=1)
    if out:
        with open(out, "w") as f:
            f.write(txt)
    print(txt)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else None)
