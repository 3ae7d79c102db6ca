"""Builds libphasesync_cuda.so in-tree with nvcc for sm_100a.

Explicit nvcc (no torch JIT cache): the .so lands next to this file, so it
travels to the GPU box with the repo snapshot.  Usage:
    python -m paper_1710_08037_b200._build [--force]
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
LIB = PKG / "libphasesync_cuda.so"
SOURCES = ["capi.cu", "prep_kernels.cu", "gram_tc.cu", "gram_f64.cu", "refine.cu", "shard_kernels.cu"]
HEADERS = ["ps_internal.h", "ptx.cuh", "epilogue.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _rpaths() -> list[str]:
    paths = ["/usr/local/cuda/lib64"]
    try:
        import nvidia  # type: ignore

        base = Path(list(nvidia.__path__)[0])
        for sub in ("cufft/lib", "cuda_runtime/lib"):
            if (base / sub).exists():
                paths.insert(0, str(base / sub))
    except Exception:
        pass
    return paths


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES + HEADERS] + [ROOT / "include" / "phasesync.h", Path(__file__)]
    return any(p.exists() and p.stat().st_mtime > t for p in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not _stale():
        return LIB
    nvcc = _nvcc()
    objdir = CSRC / "_obj"
    objdir.mkdir(exist_ok=True)
    common = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-I", str(ROOT / "include"),
              "-Xptxas", "-warn-spills"] + ARCH
    objs = []
    for src in SOURCES:
        obj = objdir / (Path(src).stem + ".o")
        cmd = [nvcc, *common, "-c", str(CSRC / src), "-o", str(obj)]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
        objs.append(str(obj))
    link = [nvcc, "-shared", *ARCH, "-o", str(LIB), *objs, "-L/usr/local/cuda/lib64", "-lcufft"]
    for rp in _rpaths():
        link += ["-Xlinker", f"-rpath={rp}"]
    if verbose:
        print(" ".join(link), flush=True)
    subprocess.run(link, check=True)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
