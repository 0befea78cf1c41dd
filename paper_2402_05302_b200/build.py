"""Build libcannikin.so in-tree: CUDA sources with nvcc for sm_100a, the host solvers with g++.

    python -m paper_2402_05302_b200.build          (or __graft_entry__.build())

The library links the NCCL that torch ships (same soname, rpath to its directory) and the static
CUDA runtime; it needs no GPU to build or to load.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(ROOT, "build", "cannikin")
LIB = os.path.join(HERE, "libcannikin.so")

CUDA_SOURCES = ["wsum_local.cu", "wsum_local_tma.cu", "twoshot.cu", "ll.cu", "ll128.cu", "nccl_path.cu", "nvls.cu", "emulate.cu", "gate.cu", "probe.cu", "green.cu",
                "api.cu"]
HOST_SOURCES = ["host_solvers.cpp", "analyzer.cpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dirs():
    site = sysconfig.get_paths()["purelib"]
    base = os.path.join(site, "nvidia", "nccl")
    inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
    if not os.path.exists(os.path.join(inc, "nccl.h")):
        raise RuntimeError(f"nccl.h not found under {inc}")
    return inc, lib


def _nvcc():
    p = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(p):
        raise RuntimeError("nvcc not found")
    return p


def _run(cmd):
    r = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
    if r.returncode != 0:
        raise RuntimeError("build failed:\n" + " ".join(cmd) + "\n" + r.stdout)
    return r.stdout


def _stale(obj, srcs):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(s) > t for s in srcs)


# CANNIKIN_NVCC_EXTRA: extra nvcc flags for build-time experiments (forces a rebuild)
EXTRA = os.environ.get("CANNIKIN_NVCC_EXTRA", "").split()


def build(verbose: bool = False, force: bool = False) -> str:
    nvcc = _nvcc()
    force = force or bool(EXTRA)
    nccl_inc, nccl_lib = _nccl_dirs()
    os.makedirs(BUILD, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    headers.append(os.path.join(INCLUDE, "cannikin.h"))
    jobs = []
    objs = []
    for src in CUDA_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        objs.append(o)
        if force or _stale(o, [s] + headers):
            jobs.append([nvcc, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xptxas", "-v",
                         "-Xcompiler", "-fPIC,-ffp-contract=off", "--expt-relaxed-constexpr",
                         *EXTRA, "-I", INCLUDE, "-I", CSRC, "-I", nccl_inc, "-c", s, "-o", o])
    for src in HOST_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        objs.append(o)
        if force or _stale(o, [s] + headers):
            jobs.append(["g++", "-O2", "-std=c++17", "-fPIC", "-ffp-contract=off", "-Wall",
                         "-I", INCLUDE, "-I", CSRC, "-c", s, "-o", o])
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        outs = list(ex.map(_run, jobs))
    if verbose:
        for o in outs:
            sys.stdout.write(o)
    if force or jobs or not os.path.exists(LIB) or _stale(LIB, objs):
        _run([nvcc, *ARCH, "-shared", "-cudart", "static", "-o", LIB, *objs,
              "-L", nccl_lib, "-l:libnccl.so.2", "-Xlinker", f"-rpath={nccl_lib}"])
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
