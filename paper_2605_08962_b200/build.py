"""Build libmuxb200.so in-tree with nvcc for sm_100a.

    python -m paper_2605_08962_b200.build [--force]

The shared library lands next to this file so that it travels with the repo
snapshot to the GPU box (git-ignored, not gpurun-ignored).
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(HERE, "libmuxb200.so")
SOURCES = ["capi.cu", "plan.cu", "lssp.cu", "reshard.cu", "segcopy.cu", "proj_gemm.cu",
           "proj_bwd.cu", "meta.cu"]
HEADERS = ["mux_common.cuh", "umma.cuh"]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
    "-I", os.path.join(ROOT, "include"),
]


def _deps():
    out = [os.path.join(ROOT, "include", "mux_b200.h")]
    for h in HEADERS:
        p = os.path.join(CSRC, h)
        if os.path.exists(p):
            out.append(p)
    return out


def _stale(target, sources):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def _compile(src):
    obj = os.path.join(OBJ, src.replace(".cu", ".o"))
    srcp = os.path.join(CSRC, src)
    if _stale(obj, [srcp] + _deps()):
        cmd = [NVCC, *FLAGS, *os.environ.get("MUX_NVCC_DEFS", "").split(), "-c", srcp,
               "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{r.stdout}\n{r.stderr}")
    return obj


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    if force:
        for f in os.listdir(OBJ):
            os.remove(os.path.join(OBJ, f))
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(_compile, SOURCES))
    if force or _stale(LIB, objs):
        cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", LIB, *objs,
               "-Xcompiler", "-fPIC"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    if verbose:
        print("built", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
