import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA kernels through the C ABI)")


@pytest.fixture(scope="session")
def oracle():
    """The reference compiled from its own sources when present (oracle/_ref),
    else the pinned restatement (oracle/_build)."""
    from oracle.oracle import Oracle, available, build
    if not available("orc"):
        build()
    return Oracle("ref") if available("ref") else Oracle("orc")


@pytest.fixture(scope="session")
def orc():
    from oracle.oracle import Oracle, available, build
    if not available("orc"):
        build()
    return Oracle("orc")
