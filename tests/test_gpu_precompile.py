"""NEXT-4 end to end on the GPU (-m gpu): an annotated CUDA program (tests/golden/compar_saxpy.cu,
two variants of one interface) is translated by comparcc, compiled with nvcc against
libcompar.so and run: the results are exact, every variant ran during calibration (1 warm-up + 3
timed each), and model mode then chose the fast variant for every remaining call."""
import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2311_03543_b200")


def test_comparcc_saxpy_end_to_end(tmp_path):
    src = os.path.join(ROOT, "tests", "golden", "compar_saxpy.cu")
    r = subprocess.run([os.path.join(PKG, "bin", "comparcc"), src, "--out", str(tmp_path)], capture_output=True,
                       text=True)
    assert r.returncode == 0, r.stderr
    assert "error" not in r.stderr
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    exe = tmp_path / "saxpy"
    cmd = [nvcc, "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-I", os.path.join(ROOT, "include"),
           "-I", str(tmp_path), str(tmp_path / "compar_saxpy.compar.cu"), str(tmp_path / "compar_saxpy.gen.cpp"),
           str(tmp_path / "compar_pc.gen.cpp"), "-L", PKG, "-lcompar", "-Xlinker", "-rpath," + PKG, "-o", str(exe)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["bad"] == 0
    assert out["calls_one_block"] == 4                 # its calibration only (W = 1 + K = 3)
    assert out["calls_grid"] == 20 - 4                 # calibration + every model-mode call
