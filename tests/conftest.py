import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) and libcqg.so")
    config.addinivalue_line("markers", "slow: large inputs")


@pytest.fixture(scope="session")
def oracle():
    from oracle.pyoracle import Oracle, build
    build()
    return Oracle()


@pytest.fixture(scope="session")
def reflib():
    from oracle.pyoracle import RefLib, have_ref
    if not have_ref():
        pytest.skip("oracle/_ref not built (reference sources absent)")
    return RefLib()


@pytest.fixture(scope="session")
def ctx():
    from paper_1101_0395_b200 import cabi
    return cabi.default_context(0)
