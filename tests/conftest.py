import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) device")


@pytest.fixture(scope="session")
def ref():
    """The reference oracle (oracle/_ref/libsbref.so): built here from /root/reference,
    prebuilt on the GPU box."""
    from oracle import oracle as O

    if not O.available():
        O.build()
    return O


@pytest.fixture(scope="session")
def pkg():
    import paper_2512_16896_b200 as P

    return P


@pytest.fixture(scope="session")
def gpu(pkg):
    if not pkg.device_available():
        pytest.fail("GPU test without a usable sm_100 device: " + pkg.lib().sb_last_error().decode())
    return pkg
