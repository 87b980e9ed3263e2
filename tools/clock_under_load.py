"""SM clock / power / throttle reasons while one variant runs back to back (~4 s), and its rate
against the ceiling scaled to that clock.  Answers: is a kernel's gap to its nominal-clock ceiling
arithmetic inefficiency, or the clock it actually runs at?  Development aid.

  python tools/clock_under_load.py VARIANT DTYPE(f32|bf16) COMPUTE(strict|tf32|bf16|split) M N K [seconds]
Ceilings (per SM per cycle): FFMA 256 FLOP (128 lanes x 2); BF16 tcgen05 8192; TF32 4096.
"""
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import pynvml  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
from gen.device import device_matrix  # noqa: E402
from paper_2311_03543_b200 import compar as cm  # noqa: E402

var, dt, comp = sys.argv[1:4]
m, n, k = (int(x) for x in sys.argv[4:7])
secs = float(sys.argv[7]) if len(sys.argv) > 7 else 4.0
compute = {"strict": cm.COMPUTE_F32_STRICT, "tf32": cm.COMPUTE_TF32, "bf16": cm.COMPUTE_BF16,
           "split": cm.COMPUTE_F32_SPLIT}[comp]
per_cycle = {"strict": 256, "bf16": 8192, "tf32": 4096, "split": 4096 / 3}[comp]

A = device_matrix(gen.TAG_A, m, k, dtype=dt)
B = device_matrix(gen.TAG_B, k, n, dtype=dt)
C = device_matrix(gen.TAG_C, m, n)
ctx = cm.Compar()
names = [v for v, _ in ctx.variants()]
d = cm.make_desc(m, n, k, A=A, B=B, C_in=C, C_out=C, alpha=1.5, beta=0.5,
                 in_dtype=cm.BF16 if dt == "bf16" else cm.F32, compute=compute,
                 variant_hint=names.index(var), stream=torch.cuda.current_stream().cuda_stream)
for _ in range(3):
    ctx.run(d)

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
sm_max = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
samples, stop = [], threading.Event()


def sampler():
    while not stop.is_set():
        samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
                        pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)))
        time.sleep(0.05)


torch.cuda.synchronize()
th = threading.Thread(target=sampler)
th.start()
t_end = time.perf_counter() + secs
ns = []
while time.perf_counter() < t_end:
    ids = [ctx.submit(d) for _ in range(4)]
    ns += [ctx.sync(t).ns for t in ids]
stop.set()
th.join()
half = samples[len(samples) // 4:]                  # the steady state (after the first quarter)
clk = statistics.median(s[0] for s in half)
pw = max(s[1] for s in half)
reasons = 0
for s in half:
    reasons |= s[2]
names_r = {pynvml.nvmlClocksThrottleReasonSwPowerCap: "sw_power_cap",
           pynvml.nvmlClocksThrottleReasonHwSlowdown: "hw_slowdown",
           pynvml.nvmlClocksThrottleReasonSwThermalSlowdown: "sw_thermal",
           pynvml.nvmlClocksThrottleReasonHwThermalSlowdown: "hw_thermal",
           pynvml.nvmlClocksThrottleReasonGpuIdle: "idle"}
t = statistics.median(ns[len(ns) // 4:])
sms = torch.cuda.get_device_properties(0).multi_processor_count
tf = 2.0 * m * n * k / t / 1e3
ceil_clk = sms * per_cycle * clk * 1e6 / 1e12
ceil_max = sms * per_cycle * sm_max * 1e6 / 1e12
print({"variant": var, "shape": [m, n, k], "compute": comp, "median_ms": t / 1e6, "tflops": round(tf, 2),
       "sm_mhz_median": clk, "sm_max_mhz": sm_max, "power_w_max": pw,
       "reasons": [v for b, v in names_r.items() if reasons & b],
       "ceiling_at_max_clock": round(ceil_max, 1), "frac_of_max_clock_ceiling": round(tf / ceil_max, 3),
       "ceiling_at_measured_clock": round(ceil_clk, 1), "frac_of_clock_scaled_ceiling": round(tf / ceil_clk, 3),
       "runs": len(ns)})
