"""Builds the in-tree engine library paper_2506_04203_b200/lib/libcascade_gpu.so.

nvcc cross-compiles sm_100a here (no GPU needed); the .so travels to the GPU
box with the repo snapshot.  All CUDA translation units are compiled with
--fmad=false and host code with -ffp-contract=off: the reference's doubles
are produced without FMA contraction (SURVEY.md hazard H2).
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIBDIR, "libcascade_gpu.so")
INCLUDE = os.path.join(ROOT, "include")
JSON_DIRS = [
    "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann",
]
STDCXX = "/usr/lib/x86_64-linux-gnu/libstdc++.so.6"

CU_SOURCES = ["k_sort.cu", "k_route.cu", "k_cost.cu", "k_solve.cu", "engine.cu"]
CPP_SOURCES = ["tracegen.cpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _json_dir() -> str:
    for d in JSON_DIRS:
        if os.path.exists(os.path.join(d, "json.hpp")):
            return d
    raise RuntimeError("nlohmann/json.hpp not found")


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        raise RuntimeError(f"build step failed: {cmd[-1]}")
    return r


def _stale(out: str, deps) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(LIBDIR, exist_ok=True)
    objdir = os.path.join(LIBDIR, "obj")
    os.makedirs(objdir, exist_ok=True)
    nvcc = _nvcc()
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    headers.append(os.path.join(INCLUDE, "cascade_gpu.h"))
    common = ["-std=c++17", "-O3", "-lineinfo", "-I", INCLUDE, "-I", CSRC,
              "-Xcompiler", "-fPIC,-ffp-contract=off,-fno-fast-math"]
    objs = []
    for src in CU_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(objdir, src + ".o")
        objs.append(o)
        if force or _stale(o, [s] + headers):
            cmd = [nvcc, *ARCH, *common, "--fmad=false", "-Xptxas", "-O3", "-c", s, "-o", o]
            if verbose:
                print(" ".join(cmd))
            _run(cmd)
    for src in CPP_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(objdir, src + ".o")
        objs.append(o)
        if force or _stale(o, [s] + headers):
            cmd = ["g++", "-std=c++17", "-O3", "-fPIC", "-ffp-contract=off", "-fno-fast-math",
                   "-I", INCLUDE, "-I", CSRC, "-I", _json_dir(), "-c", s, "-o", o]
            if verbose:
                print(" ".join(cmd))
            _run(cmd)
    if force or _stale(LIB, objs):
        link = [nvcc, *ARCH, "-shared", "-o", LIB, *objs, "-Xlinker", STDCXX]
        if verbose:
            print(" ".join(link))
        _run(link)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
