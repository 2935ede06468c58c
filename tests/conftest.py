import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) CUDA device")


@pytest.fixture(scope="session")
def gpu():
    from paper_1808_05488_b200 import cbi
    if not cbi.device_available():
        pytest.fail("GPU test selected but no sm_100 device is visible (no CPU fallback exists)")
    return cbi.Context.default()


def pytest_sessionfinish(session, exitstatus):
    """With CBG_PARITY_OUT set, write the largest max_rel_err each test observed
    (tests/oracle.py OBSERVED): the data the tolerances are set from."""
    out = os.environ.get("CBG_PARITY_OUT")
    if not out:
        return
    from tests import oracle
    if oracle.OBSERVED:
        with open(out, "w") as fh:
            json.dump(dict(sorted(oracle.OBSERVED.items())), fh, indent=1)
