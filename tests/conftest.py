import json
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
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
