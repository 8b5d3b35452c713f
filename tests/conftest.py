import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests of the CUDA path")
    config.addinivalue_line("markers", "slow: full-size configuration checks")


def golden(name):
    return np.load(os.path.join(GOLDEN, name))


@pytest.fixture(scope="session")
def gpu():
    """The engine on cuda:0.  A GPU test must never pass on a fallback:
    if the device or the library is missing the test errors loudly."""
    import paper_1801_03644_b200 as eng
    n = eng.device_count()
    if n < 1:
        raise RuntimeError("GPU test selected but no CUDA device is visible")
    return eng


@pytest.fixture(autouse=True)
def _device_checks(request):
    """With MDRQ_LIB=checked (the build with device-side bounds checks,
    common.cuh MDRQ_CHECKS) every GPU test ends with no failed check."""
    yield
    if os.environ.get("MDRQ_LIB") != "checked" or request.node.get_closest_marker("gpu") is None:
        return
    import ctypes
    from paper_1801_03644_b200 import _lib
    f = ctypes.c_uint32(0)
    _lib.check(_lib.load().mdrq_check_flags(ctypes.byref(f)))
    assert f.value & 0x80000000, "MDRQ_LIB=checked but the library was built without the checks"
    assert f.value & 0x7FFFFFFF == 0, f"device-side bounds checks failed: bits {f.value & 0x7FFFFFFF:#x}"
