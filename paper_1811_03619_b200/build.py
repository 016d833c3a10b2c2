"""Build libpipesgd.so in-tree with nvcc for sm_100a (no JIT cache, so the
shared object travels to the GPU box with the repo snapshot).

    python -m paper_1811_03619_b200.build
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
SOURCES = ["ring.cu", "star.cu", "comm.cu", "codec_kernels.cu", "calib.cu"]
OUT = os.path.join(HERE, "libpipesgd.so")
# Bounds-checked variant (tests only: PIPESGD_LIB=<this> selects it): every
# ring payload / vector / LL / flag access is checked against its buffer or
# inbox slot (csrc/ring.cu ring_access_ok) -- the pool offers no
# compute-sanitizer, so the library checks itself.
OUT_CHECKED = os.path.join(HERE, "libpipesgd_checked.so")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    # IEEE semantics are part of the contract: no fast-math, no FTZ, no FMA
    # contraction of the reference's separate multiply/subtract.
    "-ftz=false", "-prec-div=true", "-prec-sqrt=true", "-fmad=false",
    "-Xcompiler", "-fPIC", "-shared",
]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def stale(out: str = OUT) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(HERE, "..", "include", "pipesgd.h"))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build_library(force: bool = False, verbose: bool = False, checked: bool = False) -> str:
    """Compile every source to an object in parallel, then link the shared
    object (objects go to build/, git-ignored)."""
    import concurrent.futures as cf

    out = OUT_CHECKED if checked else OUT
    if not force and not stale(out):
        return out
    objdir = os.path.join(HERE, "build", "checked" if checked else "release")
    os.makedirs(objdir, exist_ok=True)
    compile_flags = [f for f in FLAGS if f != "-shared"] + (["-DPIPESGD_CHECKED"] if checked else [])
    if verbose:
        compile_flags.insert(0, "-Xptxas=-v")

    def obj(src):
        o = os.path.join(objdir, src.replace(".cu", ".o"))
        cmd = [nvcc(), *compile_flags, "-c", "-o", o, os.path.join(CSRC, src)]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
        return o

    with cf.ThreadPoolExecutor(len(SOURCES)) as pool:
        objs = list(pool.map(obj, SOURCES))
    subprocess.run([nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", out + ".tmp", *objs],
                   check=True)
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    print(build_library(force="--force" in sys.argv, verbose="-v" in sys.argv, checked="--checked" in sys.argv))
