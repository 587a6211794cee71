import os
import sys

import pytest

# fail fast instead of hanging the device if a solve ever stops converging
os.environ.setdefault("MFX_TIMEOUT_S", "60")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: full-size configuration (minutes)")


@pytest.fixture(scope="session")
def golden():
    from golden_data import load
    return load()
