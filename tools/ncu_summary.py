"""Summarise ncu artefacts into profiles/ (committed evidence).

usage:
  python tools/ncu_summary.py launches <launches.csv> <out.md>
  python tools/ncu_summary.py full <report.ncu-rep> <key> <out.json> [algorithmic_bytes] [flops]
"""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "lts__t_sector_hit_rate.pct", "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum", "smsp__inst_executed_op_tma_ld.sum",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__cluster_dim_x",
    "launch__shared_mem_per_block_dynamic",
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
         "ms": 1e-3, "msecond": 1e-3, "s": 1, "Ghz": 1e9, "Mhz": 1e6, "hz": 1}


def launches(path, out):
    per = defaultdict(lambda: [0, 0.0])
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for row in csv.DictReader(lines):
        if row.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = row["Kernel Name"].split("(")[0]
        per[name][0] += 1
        per[name][1] += float(row["Metric Value"].replace(",", "")) * SCALE.get(row["Metric Unit"], 1e-9)
    total = sum(v[1] for v in per.values())
    with open(out, "w") as f:
        f.write(f"# Launch list (ncu --metrics gpu__time_duration.sum, cold-cache, serialised)\n\nsource: `{path}`\n\n")
        f.write("| kernel | launches | total ms | share |\n|---|---|---|---|\n")
        for k, (n, t) in sorted(per.items(), key=lambda kv: -kv[1][1]):
            f.write(f"| `{k}` | {n} | {t * 1e3:.3f} | {t / total:.1%} |\n")
    print(open(out).read())


def full(path, key, out, alg_bytes=None, flops=None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    res = {}
    for vals in rows[2:3]:
        d = dict(zip(hdr, vals))
        u = dict(zip(hdr, units))
        res["kernel"] = d.get("Kernel Name", "")
        for k in KEYS:
            if k in d and d[k] not in ("", "n/a"):
                try:
                    v = float(d[k].replace(",", ""))
                except ValueError:
                    res[k] = d[k]
                    continue
                res[k] = v * SCALE.get(u[k], 1)
                res[k + ".unit"] = "base SI" if u[k] in SCALE else u[k]
    rb = res.get("dram__bytes_read.sum", 0) + res.get("dram__bytes_write.sum", 0)
    res["dram_bytes_per_launch"] = rb
    if alg_bytes:
        res["algorithmic_bytes_per_launch"] = float(alg_bytes)
        res["traffic_over_algorithmic"] = rb / float(alg_bytes)
    if flops and res.get("gpu__time_duration.sum"):
        res["tflops_under_ncu"] = float(flops) / res["gpu__time_duration.sum"] / 1e12
    res["source"] = os.path.basename(path)
    allres = {}
    if os.path.exists(out):
        with open(out) as f:
            allres = json.load(f)
    allres[key] = res
    with open(out, "w") as f:
        json.dump(allres, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(*sys.argv[2:])
