import json
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def _ensure_library() -> None:
    """Build libgpp_b200.so in-tree if it is missing (nvcc cross-compiles for
    sm_100a without a GPU), so the suite runs from a clean checkout."""
    lib = ROOT / "paper_2008_11326_b200" / "lib" / "libgpp_b200.so"
    if not lib.exists():
        import subprocess

        subprocess.run(["make", "-C", str(ROOT / "paper_2008_11326_b200" / "csrc")], check=True,
                       stdout=subprocess.DEVNULL)


def pytest_configure(config):
    _ensure_library()
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")
    config.addinivalue_line("markers", "slow: long-running (large problem sizes)")


def _gpu_available() -> bool:
    """A CUDA device node is present.  Deliberately NOT "the library loads":
    on a GPU box a missing or broken libgpp_b200.so must fail the tests."""
    import os

    return os.path.exists("/dev/nvidiactl") or os.path.exists("/dev/nvidia0")


def pytest_collection_modifyitems(config, items):
    if any("gpu" in item.keywords for item in items) and not _gpu_available():
        skip = pytest.mark.skip(reason="no CUDA device in this container")
        for item in items:
            if "gpu" in item.keywords:
                item.add_marker(skip)


def load_cases(name: str):
    return json.loads((GOLDEN / name).read_text())["cases"]


def as_complex(pairs):
    import numpy as np

    return np.array([complex(a, b) for a, b in pairs], dtype=np.complex128)
