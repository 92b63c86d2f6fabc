"""Compiles the CUDA C-ABI library libhrpb.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

Each translation unit is compiled to an object file by its own nvcc process (in parallel: the SpMM kernel
instantiations are split per TK), then the objects are linked into the shared library.
"""
from __future__ import annotations

import os
import subprocess
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "libhrpb.so")
SOURCES = ["csrc/api.cu", "csrc/build.cu", "csrc/spmm.cu", "csrc/spmm_tk16.cu", "csrc/spmm_tk32.cu",
           "csrc/spmm_sharded.cu", "csrc/reorder.cu"]
DEPS = SOURCES + ["csrc/common.cuh", "csrc/internal.h", "csrc/spmm_kernel.cuh", "../include/hrpb.h"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v"]


def stale(out: str = SO) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(os.path.join(HERE, d)) > t for d in DEPS)


def compile_so(out: str, extra: list[str] | None = None, verbose: bool = False) -> str:
    """nvcc -c every source in parallel, then nvcc -shared; `extra` flags go to every compile."""
    extra = extra or []
    with tempfile.TemporaryDirectory() as tmp:
        objs, procs = [], []
        for src in SOURCES:
            obj = os.path.join(tmp, os.path.basename(src) + ".o")
            objs.append(obj)
            procs.append((src, subprocess.Popen([NVCC, *FLAGS, *extra, "-c", "-o", obj, src], cwd=HERE,
                                                stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
        logs = []
        for src, pr in procs:
            so, se = pr.communicate()
            if pr.returncode != 0:
                raise RuntimeError(f"nvcc failed on {src}:\n{so}{se}")
            logs.append(se)
        r = subprocess.run([NVCC, *ARCH, "-shared", "-o", out, *objs, "-lcuda"], cwd=HERE, capture_output=True,
                           text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc link failed:\n" + r.stdout + r.stderr)
        if verbose:
            print("".join(logs))
    return out


def build(force: bool = False, verbose: bool = False) -> str:
    if force or stale():
        compile_so(SO, verbose=verbose)
    return SO


if __name__ == "__main__":
    print(build(force=True, verbose=True))
