"""Shared fixtures.  `-m gpu` tests need a CUDA device (B200); everything else
runs on the CPU build box.  GPU tests never read /root/reference."""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import pytest

REPO = Path(__file__).resolve().parent.parent
GOLDEN = Path(__file__).resolve().parent / "golden"
REFERENCE_SRC = Path("/root/reference/pkg/src")
if str(REPO) not in sys.path:
    sys.path.insert(0, str(REPO))
if str(GOLDEN) not in sys.path:
    sys.path.insert(0, str(GOLDEN))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (runs on the B200 box)")
    config.addinivalue_line("markers", "reference: needs /root/reference (build box only)")


def _cuda_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


def pytest_collection_modifyitems(config, items):
    has_gpu = _cuda_available()
    has_ref = REFERENCE_SRC.exists()
    skip_gpu = pytest.mark.skip(reason="no CUDA device")
    skip_ref = pytest.mark.skip(reason="/root/reference not present")
    for item in items:
        if "gpu" in item.keywords and not has_gpu:
            item.add_marker(skip_gpu)
        if "reference" in item.keywords and not has_ref:
            item.add_marker(skip_ref)


@pytest.fixture(scope="session", autouse=True)
def _built_library():
    """Build libtileprep.so in-tree if a fresh checkout lacks it (nvcc only)."""
    from paper_2603_16987_b200 import _build

    if not _build.LIB_PATH.exists():
        _build.build()
    return _build.LIB_PATH


@pytest.fixture(scope="session")
def golden():
    data = np.load(GOLDEN / "golden_v1.npz")
    meta = json.loads((GOLDEN / "golden_v1.json").read_text())
    return data, meta


@pytest.fixture(scope="session")
def reference():
    """The live reference package (build box only; tests using it carry
    @pytest.mark.reference)."""
    if not REFERENCE_SRC.exists():
        pytest.skip("/root/reference not present")
    if str(REFERENCE_SRC) not in sys.path:
        sys.path.insert(0, str(REFERENCE_SRC))
    import vlmfp

    return vlmfp
