"""Build libpaircount.so in-tree for sm_100a.

    python -m paper_1901_11204_b200.build [--force]

nvcc cross-compiles without a GPU; the .so is git-ignored but travels to the
GPU box with the gpurun snapshot.
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
SRC = HERE / "csrc" / "paircount.cu"
HDR = HERE.parent / "include" / "paircount.h"
OUT = HERE / "libpaircount.so"

NVCC_FLAGS = [
    "-O3", "-std=c++17", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC", "-shared",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (cand == "nvcc" or Path(cand).exists()):
            return cand
    return "nvcc"


CHECKED_OUT = HERE.parent / "build" / "checked" / "libpaircount.so"


def build(force: bool = False, verbose: bool = False, checked: bool = False) -> Path:
    """The shipped library, or with ``checked`` the bounds-checked debug build
    (-DPC_CHECKED=1, csrc/paircount.cu) used by scripts/sanitize_cases.py."""
    out = CHECKED_OUT if checked else OUT
    newest = max([HDR.stat().st_mtime] + [f.stat().st_mtime for f in SRC.parent.iterdir() if f.is_file()])
    if not force and out.exists() and out.stat().st_mtime >= newest:
        return out
    out.parent.mkdir(parents=True, exist_ok=True)
    tmp = out.with_suffix(".so.tmp")
    cmd = [nvcc(), *NVCC_FLAGS, *(["-Xptxas", "-v"] if verbose else []), *(["-DPC_CHECKED=1"] if checked else []),
           str(SRC), "-o", str(tmp)]
    subprocess.run(cmd, check=True)
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, checked="--checked" in sys.argv))
