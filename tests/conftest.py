import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu on the GPU box)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def C():
    import oracle
    return oracle.C()


@pytest.fixture(scope="session")
def Ref():
    import oracle
    if not oracle.ref_available():
        pytest.skip("oracle/_ref (reference build) not present")
    return oracle.Ref()


@pytest.fixture(scope="session")
def tkv():
    import paper_2510_09665_b200 as p
    p.lib()
    return p
