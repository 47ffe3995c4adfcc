import json
import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def _cuda_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _cuda_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session", autouse=True)
def built_library():
    """Build libfcg.so in-tree if it is missing or stale (nvcc cross-compiles
    without a GPU)."""
    from paper_2602_13140_b200 import _build
    if not _build.up_to_date():
        _build.build_library()
    return _build.LIB


class Golden:
    def __init__(self, name):
        self._z = np.load(GOLDEN / f"{name}.npz", allow_pickle=False)

    def __getitem__(self, k):
        return self._z[k]

    def cases(self, key="pos"):
        return sorted({k.split("/")[0] for k in self._z.files if k.endswith("/" + key)})

    def case(self, name):
        pre = name + "/"
        return {k[len(pre):]: self._z[k] for k in self._z.files if k.startswith(pre)}


@pytest.fixture(scope="session")
def golden():
    return {n: Golden(n) for n in ("neighbors", "flash", "md", "md_long")}


@pytest.fixture(scope="session")
def hashes():
    return json.loads((GOLDEN / "hashes.json").read_text())
