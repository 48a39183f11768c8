import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


def pytest_collection_modifyitems(config, items):
    if has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA GPU in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


REFERENCE_SRC = Path("/root/reference/pkg/src")
# the reference package installed unmodified by `pip install --target
# baseline/_ref` (git-ignored; it travels to the GPU box with the repo)
REFERENCE_INSTALL = ROOT / "baseline" / "_ref"


def reference_available() -> bool:
    return (REFERENCE_SRC / "sgsplat" / "render.py").exists()


def reference_package_path():
    """Directory to put on sys.path to import the reference package
    ``sgsplat`` (the unmodified install under baseline/_ref, else the
    read-only source tree in the build container), or None."""
    for p in (REFERENCE_INSTALL, REFERENCE_SRC):
        if (p / "sgsplat" / "render.py").exists():
            return p
    return None
