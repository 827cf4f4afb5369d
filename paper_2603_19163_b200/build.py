"""Builds libcugenopt.so in-tree for sm_100a (nvcc; no torch extension).

    python -m paper_2603_19163_b200.build        # or __graft_entry__.build()

Flags: -gencode arch=compute_100a,code=sm_100a, -lineinfo (ncu source page),
-fmad=false (parity: the reference rounds every product separately,
core.py:303-307, aos.py:96-100), -Xptxas -v (register / spill report).
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "lib" / "libcugenopt.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

SOURCES = [CSRC / "engine.cu", CSRC / "go_jit.cpp"]
DEPS = SOURCES + sorted((CSRC / "kernels").glob("*.cuh")) + [CSRC / "go_jit.h", CSRC / "go_drv.h",
                                                              ROOT / "include" / "cugenopt.h"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def needs_build() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    return any(p.stat().st_mtime > t for p in DEPS)


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not needs_build():
        return LIB
    LIB.parent.mkdir(parents=True, exist_ok=True)
    objs = []
    for src in SOURCES:
        obj = LIB.parent / (src.stem + ".o")
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-fmad=false", "-std=c++17",
               "-Xcompiler", "-fPIC,-O2", "-I", str(ROOT / "include"), "-I", str(CSRC),
               *os.environ.get("GO_NVCC_DEFINES", "").split(),  # diagnostic builds only
               "-c", str(src), "-o", str(obj)]
        if src.suffix == ".cu":
            cmd[1:1] = ["-Xptxas", "-v"] if verbose else []
        else:
            cmd[1:1] = ["-x", "cu"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stderr[-6000:]}")
        if verbose and r.stderr:
            print(r.stderr, file=sys.stderr)
        objs.append(str(obj))
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [NVCC, *ARCH, "-shared", "-o", str(tmp), *objs, "-lnvrtc", "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr[-4000:]}")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
