import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libfate.so")
    config.addinivalue_line("markers", "reference: needs the reference package importable")


@pytest.fixture(scope="session")
def reference():
    """The reference wfsched package (only in the build container)."""
    if not os.path.isdir(REFERENCE_SRC):
        pytest.skip("reference package not present")
    if REFERENCE_SRC not in sys.path:
        sys.path.append(REFERENCE_SRC)
    import wfsched

    return wfsched
