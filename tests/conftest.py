import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def ft():
    import paper_1710_11593_b200 as m

    return m


@pytest.fixture(scope="session")
def oracle_mod():
    import oracle

    oracle.build(reference=False)
    return oracle
