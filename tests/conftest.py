import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))  # the CPU checker (test infrastructure)

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the sm_100a C ABI)")
    config.addinivalue_line("markers", "slow: large shapes")


def pytest_collection_modifyitems(config, items):
    try:
        import torch

        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session", autouse=True)
def _built_library():
    """The control plane's first-fit planner and every kernel live in the
    in-tree C-ABI library; build it (no-op when fresh) before any test."""
    from paper_2601_06562_b200 import _build

    _build.build()


@pytest.fixture(scope="session")
def native_lib():
    from paper_2601_06562_b200 import _build, _native

    _build.build()
    return _native.load()
