"""The C ABI: the library loads without a GPU, exports every symbol the
header declares, and fails loudly (no CPU fallback) when no device exists."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "mdrq_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mdrq_[a-z_]+)\s*\(", src)))


def test_header_declares_expected_entry_points():
    from paper_1801_03644_b200 import _lib
    assert declared_functions() == sorted(_lib.EXPORTED)


def test_library_exports_every_declared_symbol():
    from paper_1801_03644_b200 import _lib
    lib = _lib.load()
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert lib.mdrq_abi_version() == 1


def test_no_cpu_fallback_without_device():
    import paper_1801_03644_b200 as eng
    if eng.device_count() > 0:
        pytest.skip("a CUDA device is present")
    with pytest.raises(RuntimeError, match="no CUDA device"):
        eng.DeviceStore(np.zeros((16, 3), np.float32))
    with pytest.raises(RuntimeError):
        eng.kernels.scan_column(np.zeros(10, np.float32), 0.0, 1.0)


def test_error_codes_map_to_python_exceptions():
    from paper_1801_03644_b200 import _lib
    lib = _lib.load()
    out = ctypes.c_void_p()
    rc = lib.mdrq_store_create(None, 0, 0, 0, 1, 0, 0, ctypes.byref(out))
    assert rc == _lib.MDRQ_EINVAL
    with pytest.raises(ValueError, match="dimensionality"):
        _lib.check(rc)


def test_shared_object_is_sm100a():
    """The cubin inside the library targets sm_100a only."""
    import shutil
    import subprocess
    from paper_1801_03644_b200 import _lib
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump unavailable")
    r = subprocess.run([exe, "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    archs = set(re.findall(r"sm_(\d+a?)", r.stdout))
    assert archs == {"100a"}, archs


def test_null_store_and_arguments_are_einval():
    """Every store entry point rejects a null store / null outputs with
    MDRQ_EINVAL instead of crashing (no device needed)."""
    from paper_1801_03644_b200 import _lib
    lib = _lib.load()
    total = ctypes.c_uint64(0)
    assert lib.mdrq_query_ids(None, None, None, 0, 0, None, None, 0, ctypes.byref(total)) == _lib.MDRQ_EINVAL
    assert lib.mdrq_query_count(None, None, None, 0, 0, None) == _lib.MDRQ_EINVAL
    assert lib.mdrq_query_ids_stream(None, None, None, None, 1, 0, None, None, None, None, None) == _lib.MDRQ_EINVAL
    assert lib.mdrq_fetch_ids(None, None, 0) == _lib.MDRQ_EINVAL
    assert lib.mdrq_last_error()
