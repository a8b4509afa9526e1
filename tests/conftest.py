import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through libprune_b200 kernels)")


def has_gpu() -> bool:
    try:
        from paper_1802_06625_b200 import _lib
        return _lib.device_count() > 0
    except Exception:  # noqa: BLE001
        return False


def pytest_collection_modifyitems(config, items):
    if has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device visible")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def golden():
    import json

    import numpy as np

    out = {}
    for name in ("dpd", "fixtures", "bypass", "policies", "motion"):
        out[name] = json.loads((GOLDEN / f"{name}.json").read_text())
    out["dpd_small"] = dict(np.load(GOLDEN / "dpd_small.npz"))
    out["bypass_small"] = dict(np.load(GOLDEN / "bypass_small.npz"))
    out["motion_small"] = dict(np.load(GOLDEN / "motion_small.npz"))
    return out
