import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
# the reference's own tests, vendored by tools/vendor_reference_tests.py, run only through
# test_gpu_reference_suite.py (they need the GPU and the `bittrain` alias of their own conftest)
collect_ignore = ["_reference"]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def oracle():
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle as _oracle  # test infrastructure only

    _oracle.build()
    return _oracle
