"""Build the CUDA engine in-tree: csrc/*.cu -> libhcnn_b200.so (sm_100a).

    python -m paper_2310_16530_b200.build [--force]

The shared library is git-ignored but travels to the GPU box with the
working tree (it is not in .gpurunignore).
"""

from __future__ import annotations

import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OUT = PKG / "libhcnn_b200.so"
SOURCES = ["ntt.cu", "ntt2.cu", "arith.cu", "capi.cu"]
NVCC_FLAGS = [
    "-O3", "-std=c++17", "--extended-lambda", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
    "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-O3",
]


def _nvcc() -> str:
    for cand in ("nvcc", "/usr/local/cuda/bin/nvcc"):
        p = shutil.which(cand) or (cand if Path(cand).exists() else None)
        if p:
            return p
    raise RuntimeError("nvcc not found")


def needs_build() -> bool:
    if not OUT.exists():
        return True
    t = OUT.stat().st_mtime
    deps = list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cuh")) + [PKG.parent / "include" / "hcnn_b200.h"]
    return any(d.stat().st_mtime > t for d in deps if d.exists())


def build(force: bool = False, verbose: bool = True) -> Path:
    if not force and not needs_build():
        return OUT
    cmd = [_nvcc(), *NVCC_FLAGS, "-o", str(OUT), *[str(CSRC / s) for s in SOURCES]]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv)
