"""Build the B200 CUDA library in-tree: paper_1803_07289_b200/libflexconv_b200.so.

nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3, one object per .cu, linked
with -shared.  Run `python -m paper_1803_07289_b200.build` (or __graft_entry__.build()).
Objects go to paper_1803_07289_b200/_build/ (git-ignored); the .so sits next to this file
so it travels to the GPU box with the snapshot.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libflexconv_b200.so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-I", INCLUDE, "-Xptxas", "-v"] + ARCH
HOST_CC = os.environ.get("FC_HOST_CC", "/usr/bin/g++")


def _sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def _headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    hs.append(os.path.join(INCLUDE, "flexconv_b200.h"))
    return hs


def _compile(src: str, verbose: bool) -> str:
    obj = os.path.join(BUILD, os.path.basename(src).replace(".cu", ".o"))
    newest_dep = max(os.path.getmtime(p) for p in [src] + _headers())
    if os.path.exists(obj) and os.path.getmtime(obj) >= newest_dep:
        return obj
    cmd = [NVCC, "-ccbin", HOST_CC, "-c", src, "-o", obj] + FLAGS
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc failed on {src}")
    log = os.path.join(BUILD, os.path.basename(src) + ".ptxas.txt")
    with open(log, "w") as fh:
        fh.write(res.stderr)
    if verbose:
        print(f"compiled {os.path.basename(src)}")
    return obj


def build(verbose: bool = True) -> str:
    os.makedirs(BUILD, exist_ok=True)
    srcs = _sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), srcs))
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        cmd = [NVCC, "-ccbin", HOST_CC, "-shared", "-o", LIB] + objs + ARCH + [
            "-lcudart", "-lcuda", "-Xlinker", "-rpath=/usr/local/cuda/lib64"]
        subprocess.check_call(cmd)
        if verbose:
            print(f"linked {LIB}")
    return LIB


if __name__ == "__main__":
    build()
