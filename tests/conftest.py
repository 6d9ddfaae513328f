import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

# peer-memory exchanges under test give up after 20 s instead of 60 s, so a broken
# peer test fails fast instead of stalling the run (EVOX_ERR_EXCHANGE)
from paper_2301_12457_b200 import evox as _evox  # noqa: E402

_evox.DEFAULT_PEER_TIMEOUT_MS = 20000


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden_dir():
    return os.path.join(ROOT, "tests", "golden")
