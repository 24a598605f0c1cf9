"""Builds the in-tree shared library ``libmgrc_gpu.so`` for sm_100a.

nvcc cross-compiles without a GPU.  The library is built in-tree so it
travels with the repository snapshot to the GPU box (it is git-ignored).
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
ROOT = PKG.parent
LIB = PKG / "libmgrc_gpu.so"

SOURCES = ["pipeline.cu", "transform.cu", "host.cpp", "capi.cpp"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "--fmad=false",                 # no FMA contraction anywhere
    "-Xcompiler", "-fPIC,-ffp-contract=off,-fvisibility=hidden",
    "-Xptxas", "-warn-spills",
]
LINK_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


FLAGS_STAMP = PKG / "build" / "extra_flags.txt"  # the MGRC_NVCC_EXTRA the library was built with


def needs_build() -> bool:
    if not LIB.exists():
        return True
    extra = os.environ.get("MGRC_NVCC_EXTRA", "")
    if (FLAGS_STAMP.read_text() if FLAGS_STAMP.exists() else "") != extra:
        return True
    t = LIB.stat().st_mtime
    deps = ([CSRC / s for s in SOURCES] + sorted(CSRC.glob("*.cuh")) + sorted(CSRC.glob("*.hpp")) +
            [ROOT / "include" / "mgrc_gpu.h", Path(__file__)])
    return any(p.stat().st_mtime > t for p in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    """Each translation unit compiles to an object in parallel (nvcc -c), then one nvcc link."""
    if not force and not needs_build():
        return LIB
    from concurrent.futures import ThreadPoolExecutor

    objdir = PKG / "build"
    objdir.mkdir(exist_ok=True)
    extra = os.environ.get("MGRC_NVCC_EXTRA", "").split()  # experiments only (e.g. -DMGRC_WARM_BITS=512)

    def compile_one(src):
        obj = objdir / (src + ".o")
        cmd = [nvcc(), *NVCC_FLAGS, *extra, "-I", str(ROOT / "include"), "-c", "-o", str(obj), str(CSRC / src)]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src} ({r.returncode}):\n{r.stdout}\n{r.stderr}")
        if verbose and r.stderr:
            print(r.stderr, file=sys.stderr)
        return obj

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [nvcc(), *LINK_FLAGS, "-o", str(tmp), *map(str, objs)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc link failed ({r.returncode}):\n{r.stdout}\n{r.stderr}")
    tmp.replace(LIB)
    FLAGS_STAMP.write_text(" ".join(extra))
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
