"""In-tree native build: libcompar.so (runtime + sm_100a kernels), gen/libcompar_gen.so, oracle.

Everything is compiled for sm_100a only (`-gencode arch=compute_100a,code=sm_100a`:
plain `-arch=sm_100a` also emits compute_100 PTX, which rejects tcgen05).  NCCL comes
from the torch wheel (one libnccl.so.2 per process), linked with an RPATH to it.
Usage: python -m paper_2311_03543_b200.build [--force]
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys
import sysconfig

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
INC = os.path.join(ROOT, "include")
BUILD = os.path.join(ROOT, "build")
LIB = os.path.join(PKG, "libcompar.so")
GEN_LIB = os.path.join(ROOT, "gen", "libcompar_gen.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    site = sysconfig.get_paths()["purelib"]
    base = os.path.join(site, "nvidia", "nccl")
    inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
    if not os.path.exists(os.path.join(inc, "nccl.h")):
        inc, lib = "/usr/include", "/usr/lib/x86_64-linux-gnu"
    return inc, lib


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("build failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
    return r.stdout + r.stderr


def build_compar(force: bool = False, verbose: bool = False) -> str:
    nccl_inc, nccl_lib = nccl_dirs()
    srcs = sorted(glob.glob(os.path.join(PKG, "csrc", "kernels", "*.cu")) +
                  glob.glob(os.path.join(PKG, "csrc", "kernels", "*.cpp")) +
                  glob.glob(os.path.join(PKG, "csrc", "runtime", "*.cpp")))
    headers = (glob.glob(os.path.join(PKG, "csrc", "*", "*.h")) + glob.glob(os.path.join(PKG, "csrc", "*", "*.cuh")) +
               [os.path.join(INC, "compar.h")])
    os.makedirs(BUILD, exist_ok=True)
    flags = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
                    "-I", INC, "-I", nccl_inc, "-Xptxas", "-v" if verbose else "-O3"]
    jobs = []
    objs = []
    for s in srcs:
        o = os.path.join(BUILD, os.path.basename(s) + ".o")
        objs.append(o)
        if force or _stale(o, [s] + headers):
            jobs.append([NVCC] + flags + ["-c", s, "-o", o])
    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        for out in ex.map(_run, jobs):
            if verbose and out:
                print(out)
    if force or jobs or _stale(LIB, objs):
        _run([NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", LIB + ".tmp"] + objs +
             ["-L", nccl_lib, "-l:libnccl.so.2", "-Xlinker", "-rpath," + nccl_lib])
        os.replace(LIB + ".tmp", LIB)
    return LIB


def build_gen(force: bool = False) -> str:
    src = os.path.join(ROOT, "gen", "gen.cu")
    if force or _stale(GEN_LIB, [src, os.path.join(INC, "compar_gen.h")]):
        _run([NVCC] + ARCH + ["-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-shared", "-cudart", "static",
                              "-I", INC, "-o", GEN_LIB + ".tmp", src])
        os.replace(GEN_LIB + ".tmp", GEN_LIB)
    return GEN_LIB


COMPARCC = os.path.join(PKG, "bin", "comparcc")


def build_precompiler(force: bool = False) -> str:
    """comparcc, the #pragma compar pre-compiler (host C++)."""
    src = os.path.join(PKG, "csrc", "precompiler", "comparcc.cpp")
    if force or _stale(COMPARCC, [src]):
        os.makedirs(os.path.dirname(COMPARCC), exist_ok=True)
        _run(["g++", "-O2", "-std=c++17", "-Wall", "-Wextra", "-o", COMPARCC + ".tmp", src])
        os.replace(COMPARCC + ".tmp", COMPARCC)
    return COMPARCC


def build_all(force: bool = False, verbose: bool = False):
    """Product library + the input-generator twin + the pre-compiler.  (The oracle is compiled by
    __graft_entry__.build() / the tests; the product package never touches oracle/.)"""
    return [build_compar(force, verbose), build_gen(force), build_precompiler(force)]


if __name__ == "__main__":
    for p in build_all(force="--force" in sys.argv, verbose="-v" in sys.argv):
        print(p)
