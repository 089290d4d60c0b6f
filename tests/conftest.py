import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU; run with -m gpu")
    config.addinivalue_line("markers", "ref: needs the reference simulator build oracle/_ref")


@pytest.fixture(scope="session")
def ctx():
    import paper_1606_08150_b200 as dpc
    c = dpc.Context(0)  # fails loudly on a GPU box without a usable device
    yield c
    c.close()


@pytest.fixture(scope="session")
def orc():
    from tests import _oracle
    return _oracle.Oracle()
