import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running (config 5 setup etc.)")


def _has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


HAS_GPU = _has_gpu()


def pytest_collection_modifyitems(config, items):
    if HAS_GPU:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def restatement():
    from oracle import checkers as O

    return O.Restatement()


@pytest.fixture(scope="session")
def golden():
    from tests.golden_io import load_golden

    return load_golden


@pytest.fixture(scope="session")
def reference():
    """The reference library built in place (oracle/_ref); skips when absent."""
    from oracle import checkers as O

    try:
        return O.Reference()
    except O.ReferenceUnavailable as e:  # pragma: no cover
        pytest.skip(str(e))
