import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def port():
    import oracle
    return oracle.port()


@pytest.fixture(scope="session")
def ref():
    import oracle
    if not (os.path.exists(oracle.REF_SO) or os.path.isdir(oracle.REF_SRC)):
        pytest.skip("reference oracle not available")
    return oracle.ref()


GOLDEN = os.path.join(ROOT, "tests", "golden")
