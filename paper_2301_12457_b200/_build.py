"""In-tree build of libevox.so for sm_100a (nvcc cross-compiles without a GPU).

The .so is git-ignored but travels to the GPU box with the gpurun snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(PKG, "build")
LIB = os.path.join(PKG, "libevox.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC,-Wall", "-I", INCLUDE, "-I", CSRC,
          "-I", "/usr/include"]
SOURCES = ["pso_kernels.cu", "cso_kernels.cu", "de_kernels.cu", "common_kernels.cu", "evox_api.cpp",
           "nccl_dl.cpp"]
HEADERS = ["evox_device.cuh", "row_engine.cuh", "evox_internal.h", "nccl_dl.h"]


def _newest_input() -> float:
    paths = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(INCLUDE, "evox.h"),
                                                                    __file__]
    return max(os.path.getmtime(p) for p in paths)


def _compile(src: str, verbose: bool, bdir: str = BUILD, dflags=()) -> str:
    obj = os.path.join(bdir, os.path.splitext(src)[0] + ".o")
    lang = ["-x", "cu"] if src == "evox_api.cpp" else []  # includes the device header
    cmd = [NVCC, *ARCH, *COMMON, *dflags, *lang, "-c", os.path.join(CSRC, src), "-o", obj]
    if src.endswith(".cu"):
        cmd += ["-Xptxas", "-v"] if verbose else []
    subprocess.check_call(cmd)
    return obj


def build(force: bool = False, verbose: bool = False, defines=(), out: str = LIB) -> str:
    """Build libevox.so; `defines` (e.g. ["EVOX_U=2"]) produce tuning variants at `out`."""
    if not force and not defines and os.path.exists(out) and os.path.getmtime(out) >= _newest_input():
        return out
    bdir = BUILD if not defines else BUILD + "_" + "_".join(d.replace("=", "") for d in defines)
    os.makedirs(bdir, exist_ok=True)
    dflags = [f"-D{d}" for d in defines]
    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose, bdir, dflags), SOURCES))
    tmp = out + f".tmp{os.getpid()}"
    subprocess.check_call([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs, "-ldl",
                           "-lpthread"])
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
