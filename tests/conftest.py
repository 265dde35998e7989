import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

REF_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 GPU (runs through libmgrgpu.so)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def ncpflow():
    """The reference package, importable only in the build container."""
    if not os.path.isdir(REF_SRC):
        pytest.skip("reference not mounted (GPU box)")
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import ncpflow as m  # noqa: F401
    import ncpflow.amg, ncpflow.mgr, ncpflow.krylov, ncpflow.sparse  # noqa: E401,F401
    return m


@pytest.fixture(scope="session")
def gpu():
    from paper_1801_08464_b200 import _lib
    return _lib.ctx()
