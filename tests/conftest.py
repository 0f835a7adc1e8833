import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libscmoe.so")
    config.addinivalue_line("markers", "slow: long-running GPU case")


@pytest.fixture(scope="session")
def orc():
    import _oracle
    return _oracle.orc()


@pytest.fixture(scope="session")
def ref():
    import _oracle
    if not _oracle.ref_available():
        pytest.skip("oracle/_ref not built (no /root/reference and no prebuilt .so)")
    return _oracle.ref()


@pytest.fixture(scope="session")
def scmoe():
    """The product package, with its CUDA library built and a device present."""
    import paper_2509_01322_b200 as P
    from paper_2509_01322_b200 import build as B
    B.build()
    P.default_context()  # raises if no B200: GPU tests must not silently pass
    return P
