"""Build libsgs.so (sm_100a) in-tree with nvcc.

The shared library is the product: every render, sort and gradient in this
package runs through it.  It is compiled from ``csrc/*.cu`` with
``-gencode arch=compute_100a,code=sm_100a -lineinfo`` and written to
``paper_2509_07021_b200/_lib/libsgs.so`` so that it travels with the source
tree to the GPU box (the .so is git-ignored, not gpurun-ignored).
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
CSRC = PKG_DIR / "csrc"
LIB_DIR = PKG_DIR / "_lib"
LIB_PATH = LIB_DIR / "libsgs.so"
SOURCES = ["api.cu", "preprocess.cu", "binning.cu", "raster.cu", "preprocess_bwd.cu", "loss.cu", "select.cu", "compact.cu"]
HEADERS = ["common.cuh", "sgs_geom.h", "sort.cuh"]
ARCH_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-shared",
              "--expt-relaxed-constexpr"]


def nvcc_path() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; cannot build libsgs.so")


def _stale() -> bool:
    if not LIB_PATH.exists():
        return True
    t = LIB_PATH.stat().st_mtime
    deps = [CSRC / s for s in SOURCES + HEADERS] + [PKG_DIR.parent / "include" / "sgs.h"]
    return any(p.stat().st_mtime > t for p in deps if p.exists())


def build_lib(force: bool = False, verbose: bool = False) -> Path:
    """Compile libsgs.so if missing or older than its sources."""
    if not force and not _stale():
        return LIB_PATH
    LIB_DIR.mkdir(exist_ok=True)
    tmp = LIB_PATH.with_suffix(".so.tmp")
    cmd = [nvcc_path(), *NVCC_FLAGS, *ARCH_FLAGS, "-o", str(tmp),
           *[str(CSRC / s) for s in SOURCES]]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{res.stderr[-4000:]}")
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


if __name__ == "__main__":
    print(build_lib(force="--force" in sys.argv, verbose=True))
