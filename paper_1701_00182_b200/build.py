"""In-tree build of libacrgpu.so (sm_100a) with nvcc.  No JIT cache: the built
.so lives next to this file and travels with the repo snapshot."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libacrgpu.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "--expt-relaxed-constexpr"]
SOURCES = ["structure.cpp", "kernels.cu", "krylov.cu", "engine.cu"]
HEADERS = sorted(f for f in os.listdir(CSRC) if f.endswith((".hpp", ".cuh"))) + [os.path.join("..", "..", "include", "acrgpu.h")]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False, defines=(), lib: str | None = None) -> str:
    """Compile csrc/ into LIB (or `lib`, with extra -D `defines`: kernel-variant A/B builds,
    selected at run time by ACRGPU_LIB)."""
    objdir = os.path.join(HERE, "build" if not defines else "build_" + "_".join(d.replace("=", "") for d in defines))
    out = lib or LIB
    os.makedirs(objdir, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS]
    objs = []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(objdir, src + ".o")
        objs.append(o)
        if force or _stale(o, [s] + hdrs):
            dflags = [f"-D{d}" for d in defines]
            cmd = [NVCC, *ARCH, *FLAGS, *dflags, "-c", s, "-o", o]
            if src.endswith(".cpp"):
                cmd = [NVCC, *ARCH, *FLAGS, *dflags, "-x", "c++", "-c", s, "-o", o]
            if verbose:
                print(" ".join(cmd), file=sys.stderr)
            subprocess.run(cmd, check=True)
    if force or _stale(out, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", out, *objs, "-cudart=static"]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
    return out


if __name__ == "__main__":
    print(build(verbose=True, force="--force" in sys.argv))
