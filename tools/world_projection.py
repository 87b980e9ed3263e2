"""Inputs of the multi-GPU projection, measured on ONE B200, and the projection.

Config 4 (32768^3 BF16, C = 1.5AB + 0.5C) row panels for P = 1, 2, 4, 8 (rows 32768 / P):
  * full:  the panel GEMM (wide pair kernel) on all SMs;
  * res:   the same on num_sms - 4 SMs (COMPAR_NUM_SMS; the SMs an NCCL broadcast with
           maxCTAs = 4 occupies);
  * loop:  the world pipeline in loopback (COMPAR_BCAST_LOOPBACK=1): B packed into 64 slabs by the
           copy engine, "broadcast" by D2D copies, the fused flag-waiting launch consuming them in
           geometric column groups — the receiver's code path, with a very fast broadcast.
The three are interleaved round by round (3 rounds x 3 launches, medians) so that they see the
same power-capped clocks.
Projection for a broadcast bandwidth BW (unmeasured here: one GPU per gpurun):
  receiver = first slab (K x 512 x 2 B) / BW + the fused GEMM (loop), if BW keeps ahead of its
             consumption (2 GiB / GEMM time), else broadcast time + one slab's GEMM;
  root     = GEMM on num_sms - 4 SMs while the broadcast runs, then on all SMs (helper launch);
  E_P      = T_1 / (P * max(root, receiver)).
usage: python tools/world_projection.py [out.json]
"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import gen  # noqa: E402
from gen.device import fill  # noqa: E402
from paper_2311_03543_b200 import compar as cm  # noqa: E402

S = 32768


def ctx_with(env):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return cm.Compar(bcast_chunks=8)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def measure(P, sms, rounds=3, reps=3):
    """full / res / loop for one panel size, interleaved round by round (same power state)."""
    rows = S // P
    modes = {"full": ({}, 0), "res": ({"COMPAR_NUM_SMS": str(sms - 4)}, 0), "loop": ({"COMPAR_BCAST_LOOPBACK": "1"}, 1)}
    ctxs = {m: ctx_with(env) for m, (env, _) in modes.items()}
    sp = torch.cuda.current_stream().cuda_stream
    A = torch.empty((rows, S), dtype=torch.bfloat16, device="cuda")
    B = torch.empty((S, S), dtype=torch.bfloat16, device="cuda")
    C = torch.empty((rows, S), dtype=torch.float32, device="cuda")
    fill(A.data_ptr(), "bf16", rows, S, S, gen.TAG_A, stream=sp)
    fill(B.data_ptr(), "bf16", S, S, S, gen.TAG_B, stream=sp)
    fill(C.data_ptr(), "f32", rows, S, S, gen.TAG_C, stream=sp)
    descs = {}
    for m, (env, world) in modes.items():
        names = [v for v, _ in ctxs[m].variants()]
        descs[m] = cm.make_desc(rows, S, S, A=A, B=B, C_in=C, C_out=C, alpha=1.5, beta=0.5, in_dtype=cm.BF16,
                                compute=cm.COMPUTE_BF16, stream=sp, world=world,
                                variant_hint=names.index("tc_bf16_2sm_w"))
        ctxs[m].run(descs[m])
    samples = {m: [] for m in modes}
    for r in range(rounds):
        for m in (list(modes)[r % 3:] + list(modes)[:r % 3]):
            samples[m] += [ctxs[m].run(descs[m]) for _ in range(reps)]
    out = {"rows": rows}
    for m in modes:
        rs = samples[m]
        out[m] = {"kernel_ms": statistics.median(x.ns for x in rs) / 1e6,
                  "total_ms": statistics.median(x.total_ns for x in rs) / 1e6,
                  "bcast_ms": statistics.median(x.bcast_ns for x in rs) / 1e6}
        ctxs[m].terminate()
    del A, B, C
    torch.cuda.empty_cache()
    return out


def project(t1, full, res, loop, bw_gbs, nslab=64):
    bbytes = 2.0 * S * S
    tb = bbytes / (bw_gbs * 1e9) * 1e3                 # ms
    first = tb / nslab
    consume = bbytes / (loop * 1e-3) / 1e9             # GB/s the receiver's fused GEMM reads B at
    receiver = (first + loop) if bw_gbs >= consume else (tb + loop / nslab)
    root = res if tb >= res else tb + (1.0 - tb / res) * full
    return max(root, receiver), root, receiver


def main(out):
    torch.cuda.set_device(0)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    meas = {}
    for P in (1, 2, 4, 8):
        meas[P] = measure(P, sms)
        print(P, json.dumps(meas[P]), flush=True)
    t1 = meas[1]["full"]["kernel_ms"]
    proj = {}
    for bw in (150, 200, 300, 400, 600, 900):
        row = {}
        for P in (2, 4, 8):
            tp, root, rec = project(t1, meas[P]["full"]["kernel_ms"], meas[P]["res"]["kernel_ms"],
                                    meas[P]["loop"]["kernel_ms"], bw)
            row[P] = {"T_P_ms": tp, "root_ms": root, "receiver_ms": rec, "E_P": t1 / (P * tp)}
        proj[bw] = row
        print(f"BW {bw} GB/s: " + "  ".join(f"E{P}={row[P]['E_P']:.3f}" for P in (2, 4, 8)), flush=True)
    res = {"what": __doc__.strip().splitlines()[0], "sms": sms, "measured": meas, "projection_by_bcast_gbs": proj}
    if out:
        with open(out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else None)
