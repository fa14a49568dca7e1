import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

REF_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")
    config.addinivalue_line("markers", "slow: takes more than a few seconds on CPU")


@pytest.fixture(scope="session")
def reference():
    """The reference package, importable only in the build container."""
    if not os.path.isdir(REF_SRC):
        pytest.skip("reference not present (GPU box)")
    if REF_SRC not in sys.path:
        sys.path.append(REF_SRC)
    import seethrough
    return seethrough
