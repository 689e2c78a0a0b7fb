"""Build the CUDA shared library in-tree (sm_100a only).

    python -m paper_1807_10749_b200.build

Produces ``paper_1807_10749_b200/libgridsim_b200.so`` with nvcc
(``-gencode arch=compute_100a,code=sm_100a -lineinfo``, static cudart so the
library does not depend on which CUDA runtime the host process loaded).
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT = os.path.join(PKG, "libgridsim_b200.so")
SOURCES = ["engine.cu", "pass_kernels.cu", "jit.cu", "sampler.cu"]
DEPS = ["engine.cu", "pass_kernels.cu", "jit.cu", "sampler.cu", "jit.hpp", "jitgen.inc", "kernels.cuh", "program.hpp",
        "pass_kernel.cuh", "pass_kernel.h", "pass_types.h"]

NVCC_FLAGS = [
    "-O3",
    "-std=c++17",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo",
    "-Xcompiler", "-fPIC",
    "-Xcompiler", "-O2",
    "-Xptxas", "-v",
]
LINK_FLAGS = ["-shared", "-cudart", "static", "-gencode", "arch=compute_100a,code=sm_100a", "-ldl"]


def nvcc_path() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, d) for d in DEPS] + [os.path.join(ROOT, "include", "gridsim_b200.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return OUT
    objdir = os.path.join(ROOT, "build", "obj")
    os.makedirs(objdir, exist_ok=True)
    nvcc = nvcc_path()
    procs = []
    for src in SOURCES:
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        # GS_EXTRA_NVCC: extra defines for A/B experiments (e.g. -DGS_PROJ_PREFETCH_G=0)
        cmd = [nvcc, *NVCC_FLAGS, *os.environ.get("GS_EXTRA_NVCC", "").split(), "-c", "-o", obj,
               os.path.join(CSRC, src)]
        procs.append((src, obj, subprocess.Popen(cmd, cwd=CSRC, stdout=subprocess.PIPE,
                                                 stderr=subprocess.PIPE, text=True)))
    objs = []
    for src, obj, p in procs:
        out, err = p.communicate()
        if p.returncode != 0:
            sys.stderr.write(out + err)
            raise RuntimeError(f"nvcc failed on {src}")
        if verbose:
            sys.stderr.write(err)
        objs.append(obj)
    cmd = [nvcc, *LINK_FLAGS, "-o", OUT + ".tmp", *objs]
    res = subprocess.run(cmd, cwd=CSRC, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc link failed for libgridsim_b200.so")
    os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
