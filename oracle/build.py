"""TEST INFRASTRUCTURE: compile the oracle's C restatement (ref_kernels.c)
into oracle/liboracle.so with gcc (-fopenmp).  Not part of the product."""

from __future__ import annotations

import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
SRC = HERE / "ref_kernels.c"
OUT = HERE / "liboracle.so"


def build(force: bool = False) -> Path:
    if not force and OUT.exists() and OUT.stat().st_mtime > SRC.stat().st_mtime:
        return OUT
    subprocess.run(["gcc", "-O3", "-march=x86-64-v2", "-fopenmp", "-fPIC", "-shared", "-o", str(OUT), str(SRC)],
                   check=True)
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv)
