"""Sort interface throughput on one B200: each variant over n, FP32 keys uniform
in bits (special values included), CUDA-event time of the sort task (median of R), Gkeys/s and
the HBM bandwidth it implies at the radix sort's compulsory traffic (4 B/key histogram read +
4 passes x 8 B/key = 36 B/key) and at the one-pass floor (8 B/key).
usage: python tools/sort_bench.py [out.json]
"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2311_03543_b200 import compar as cm  # noqa: E402

R = 10


def main(out):
    torch.cuda.set_device(0)
    ctx = cm.Compar()
    names = [n for n, _ in ctx.variants()]
    res = []
    for n in [1 << 10, 1 << 12, 1 << 14, 1 << 16, 1 << 18, 1 << 20, 1 << 22, 1 << 24, 1 << 26, 1 << 28]:
        x = torch.randint(-2 ** 31, 2 ** 31 - 1, (n,), dtype=torch.int32, device="cuda").view(torch.float32)
        t = torch.empty_like(x)
        row = {"n": n}
        for name in ("sort_bitonic", "sort_radix"):
            if name == "sort_bitonic" and n > 16384:
                continue
            ts = []
            for _ in range(R + 1):
                t.copy_(x)
                ts.append(ctx.sort(t, key_type=cm.KEY_F32, variant_hint=names.index(name),
                                   stream=torch.cuda.current_stream().cuda_stream).ns)
            med = statistics.median(ts[1:])
            row[name] = {"us": med / 1e3, "gkeys_s": n / med, "gbs_at_36B": 36 * n / med,
                         "gbs_at_8B": 8 * n / med}
        res.append(row)
        print(json.dumps(row), flush=True)
        del x, t
        torch.cuda.empty_cache()
    ctx.terminate()
    if out:
        with open(out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else None)
