"""The built library really contains Blackwell-native code (-m "not gpu"; SURVEY §5 aux item).

`cuobjdump -sass libcompar.so` is split per kernel and each kernel family must contain its
defining instructions (B200_PROFILING.md SASS mnemonics):
  * tcgen05 kernels: UTCHMMA (tcgen05.mma; .2CTA for the CTA-pair forms), UTMALDG (TMA loads),
    LDTM (tcgen05.ld from TMEM); the TMA-epilogue pair / wide kernels also UTMASTG (TMA stores);
    the wide kernel's row-major instantiations the 3-D slab-packed B loads (UTMALDG.3D.2CTA);
  * FFMA variants: FFMA2 (sm_100 paired FMA; every simt_f32 and tma_f32 instantiation).
"""
import os
import re
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2311_03543_b200", "libcompar.so")


@pytest.fixture(scope="module")
def kernels():
    if not shutil.which("cuobjdump") and not os.path.exists("/usr/local/cuda/bin/cuobjdump"):
        pytest.skip("cuobjdump not available")
    if not os.path.exists(LIB):
        pytest.skip("libcompar.so not built")
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    sass = subprocess.run([exe, "-sass", LIB], capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in sass or "SM100" in sass.upper()
    out = {}
    for sec in re.split(r"\n\s*Function : ", sass)[1:]:
        mangled = sec.split("\n", 1)[0].strip()
        name = subprocess.run(["c++filt", mangled], capture_output=True, text=True).stdout.strip() or mangled
        out[name] = set(re.findall(r"\b([A-Z][A-Z0-9_]*(?:\.[A-Z0-9_]+)*)\b", sec))
    return out


def family(kernels, tag):
    got = {n: ops for n, ops in kernels.items() if tag in n}
    assert got, f"no {tag} kernel in libcompar.so"
    return got


def has(ops, prefix):
    return any(o == prefix or o.startswith(prefix + ".") for o in ops)


def test_tcgen05_one_sm_kernels(kernels):
    for tag in ("tc_gemm_kernel<", "tc_gemm_ck_kernel<"):
        for n, ops in family(kernels, tag).items():
            assert has(ops, "UTCHMMA") and has(ops, "UTMALDG") and has(ops, "LDTM"), n


def test_tcgen05_pair_kernels(kernels):
    for tag in ("tc_gemm_2sm_kernel<", "tc_gemm_2sm_mc_kernel<", "tc_gemm_2sm_wide_kernel<"):
        for n, ops in family(kernels, tag).items():
            assert "UTCHMMA.2CTA" in ops and has(ops, "LDTM"), n
            assert any(o.startswith("UTMALDG") and o.endswith("2CTA") for o in ops), n
            if tag != "tc_gemm_2sm_kernel<":          # TMA epilogue
                assert has(ops, "UTMASTG"), n
    for n, ops in family(kernels, "tc_gemm_2sm_wide_kernel<").items():
        if ", false>" in n:                           # row-major B: 3-D slab-packed loads (world mode)
            assert "UTMALDG.3D.2CTA" in ops, n


def test_ffma_kernels_use_ffma2(kernels):
    for n, ops in family(kernels, "simt_f32_kernel<").items():
        assert "FFMA2" in ops, n
    for n, ops in family(kernels, "tma_f32_kernel<").items():
        assert "FFMA2" in ops and has(ops, "UTMALDG"), n
