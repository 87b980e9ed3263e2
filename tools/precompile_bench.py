"""comparcc throughput (NEXT-4 measurement): a synthetic annotated source of L lines (interfaces
with CUDA variants and parameters, call sites, passthrough code), translated end to end (parse,
analyze, call sites, all output files); median wall time of R runs -> lines/s.
usage: python tools/precompile_bench.py [lines] [out.json]"""
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
COMPARCC = os.path.join(ROOT, "paper_2311_03543_b200", "bin", "comparcc")


def synth(lines):
    out = ["#include <cstdio>", "#pragma compar include"]
    n_if = 0
    while len(out) < lines - 4:
        i = n_if
        n_if += 1
        out += [f"#pragma compar method_declare interface(op{i}) target(CUDA) name(op{i}_a)",
                f"#pragma compar parameter name(y) type(float) size(n) access_mode(readwrite)",
                f"#pragma compar parameter name(x) type(float) size(n, m) access_mode(read)",
                f"#pragma compar parameter name(n) type(int) access_mode(read)",
                f"#pragma compar parameter name(m) type(int) access_mode(read)",
                f"#pragma compar method_declare interface(op{i}) target(CUBLAS) name(op{i}_b)"]
        out += [f"static int helper{i}_{j}(int v) {{ return v * {j} + 1; }}" for j in range(10)]
        out += [f"void use{i}(float *y, float *x, int n, int m) {{", f"    op{i}(y, x, n, m);  // call", "}"]
    out += ["int main() {", "    #pragma compar initialize", "    #pragma compar terminate", "}"]
    return "\n".join(out) + "\n", n_if


if __name__ == "__main__":
    lines = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
    text, n_if = synth(lines)
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "big.cu")
        with open(src, "w") as f:
            f.write(text)
        ts = []
        for _ in range(5):
            t0 = time.perf_counter()
            r = subprocess.run([COMPARCC, src, "--out", d], capture_output=True, text=True)
            ts.append(time.perf_counter() - t0)
            assert r.returncode == 0, r.stderr[-2000:]
        n_files = len([x for x in os.listdir(d) if x.endswith(".gen.cpp")])
    med = statistics.median(ts)
    res = {"lines": text.count("\n"), "interfaces": n_if, "glue_files": n_files, "median_s": med,
           "lines_per_s": text.count("\n") / med, "runs": ts}
    print(json.dumps(res))
    if len(sys.argv) > 2:
        with open(sys.argv[2], "w") as f:
            json.dump(res, f, indent=1)
