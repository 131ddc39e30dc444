import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

# The reference scheduler package ``wfsched`` -- the API this repository is a
# drop-in for.  ``baseline/_ref`` holds the reference installed unmodified
# (pip --target, git-ignored, travels to the GPU box with the snapshot); the
# build container also has the read-only source tree.
REFERENCE_SRC = "/root/reference/pkg/src"
REFERENCE_INSTALL = os.path.join(ROOT, "baseline", "_ref")
for _p in (REFERENCE_INSTALL, REFERENCE_SRC):
    if os.path.isdir(os.path.join(_p, "wfsched")):
        if _p not in sys.path:
            sys.path.append(_p)
        break


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libfate.so")
    config.addinivalue_line("markers", "reference: needs the reference package importable")


@pytest.fixture(scope="session")
def reference():
    """The reference wfsched package."""
    try:
        import wfsched
    except ImportError:
        pytest.skip("reference package not importable")
    return wfsched
