import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu)")


@pytest.fixture(scope="session")
def port():
    from oracle import oracle as O
    return O.port()


@pytest.fixture(scope="session")
def ref():
    from oracle import oracle as O
    if not os.path.exists(O.REF_PATH):
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return O.ref()


@pytest.fixture(scope="session")
def sd():
    import paper_2206_11664_b200 as S
    return S
