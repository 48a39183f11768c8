"""Build a libsgs variant with extra -D flags into _var/libsgs_<name>.so.
  python scratch/variant.py NAME [-DFOO=1 ...]"""
import subprocess, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2509_07021_b200 import _build as B
name, flags = sys.argv[1], sys.argv[2:]
out = B.PKG_DIR.parent / "_var" / f"libsgs_{name}.so"
cmd = [B.nvcc_path(), *B.NVCC_FLAGS, *B.ARCH_FLAGS, *flags, "-o", str(out), *[str(B.CSRC / s) for s in B.SOURCES]]
r = subprocess.run(cmd, capture_output=True, text=True)
print(name, "rc", r.returncode, r.stderr[-2000:])
