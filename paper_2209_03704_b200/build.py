"""Builds the sm_100a shared library in-tree (no JIT cache, no pip install).

    python -m paper_2209_03704_b200.build        # or __graft_entry__.build()

Each csrc/*.cu is compiled to an object in parallel with
``nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3`` and linked into
``paper_2209_03704_b200/libsegconv_b200.so`` (static cudart, no torch types).
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(PKG, "libsegconv_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-I" + os.path.join(ROOT, "include"), "-I" + CSRC]


def _compile(src: str, verbose: bool) -> str:
    obj = os.path.join(BUILD, os.path.basename(src) + ".o")
    deps = [src] + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + \
        [os.path.join(ROOT, "include", "segconv_b200.h")]
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(d) for d in deps):
        return obj
    cmd = [NVCC, *ARCH, *FLAGS, "-Xptxas", "-v" if verbose else "-O3", "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed on {src}:\n{r.stderr}")
    if verbose:
        sys.stderr.write(r.stderr)
    return obj


def build(verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), srcs))
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", LIB, *objs, "-lcuda", "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    build_cli()
    return LIB


CLI_SRC = os.path.join(ROOT, "tools", "segconv_b200.cpp")
CLI = os.path.join(ROOT, "tools", "segconv_b200")


def build_cli() -> str:
    """The command-line caller (tools/segconv_b200.cpp: verify / bench / apply
    over the drop-in C++ API), linked against the in-tree library; the
    reference's bit-for-bit default math (EXACT), as its CLI's ops are."""
    if os.path.exists(CLI) and os.path.getmtime(CLI) >= max(
            os.path.getmtime(p) for p in (CLI_SRC, LIB, os.path.join(ROOT, "include", "segconv_b200.hpp"))):
        return CLI
    cmd = ["g++", "-std=c++17", "-O2", "-DSEGCONV_B200_DEFAULT_MATH=SEGCONV_MATH_EXACT",
           "-I" + os.path.join(ROOT, "include"), "-I/usr/local/cuda/include", CLI_SRC, "-o", CLI,
           "-L" + PKG, "-lsegconv_b200", "-L/usr/local/cuda/lib64", "-lcudart", "-Wl,-rpath," + PKG,
           "-Wl,-rpath,/usr/local/cuda/lib64"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"CLI build failed:\n{r.stderr}")
    return CLI


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
