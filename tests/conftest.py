import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through libpasgal_bcc.so on cuda:0)")
    config.addinivalue_line("markers", "slow: large parity sizes (BASELINE configs)")


@pytest.fixture(scope="session", autouse=True)
def _oracle_built():
    import oracle

    oracle.build()
