"""Build the in-tree CUDA library ``libpzx_gpu.so`` for sm_100a.

The product has one native artefact: ``paper_2403_06777_b200/libpzx_gpu.so``
(C ABI in ``include/pzx_gpu.h``). It is built in-tree so that it travels with
the repository snapshot to the GPU box; nothing is installed into site-packages.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INC = os.path.join(ROOT, "include")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libpzx_gpu.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

SOURCES_CU = ["pzx_kernels.cu", "pzx_microbench.cu"]
SOURCES_CPP = ["pzx_host.cpp", "pzx_group.cpp", "pzx_reduce.cpp"]
HEADERS = ["pzx_internal.h", "pzx_math.hpp", "pzx_classes.h", "pzx_slice_dispatch.inc"]


def _run(cmd: list[str]) -> None:
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("build step failed: " + " ".join(cmd))


def _stale(out: str, deps: list[str]) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    from . import gen_slice_ops  # regenerate the bit-sliced PTX dispatch if its generator changed
    gen_slice_ops.main()
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(INC, "pzx_gpu.h")]
    objs = []
    for src in SOURCES_CU:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        if force or _stale(o, [s] + hdrs):
            _run([NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xptxas", "-v" if verbose else "-O3",
                  "-Xcompiler", "-fPIC", "-I", INC, "-I", CSRC, "-c", s, "-o", o])
        objs.append(o)
    for src in SOURCES_CPP:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        if force or _stale(o, [s] + hdrs):
            _run(["g++", "-std=gnu++17", "-O2", "-fPIC", "-Wall", "-Wextra", "-I", INC, "-I", CSRC,
                  "-I", "/usr/local/cuda/include", "-c", s, "-o", o])
        objs.append(o)
    if force or _stale(LIB, objs):
        _run([NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-cudart", "static"])
    return LIB


if __name__ == "__main__":
    sys.path.insert(0, ROOT)
    from paper_2403_06777_b200 import build as _b
    print(_b.build(force="--force" in sys.argv, verbose="-v" in sys.argv))
