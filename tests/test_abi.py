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
    return sorted(set(re.findall(r"\b(mdrq_[a-z0-9_]+)\s*\(", src)))


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
    assert lib.mdrq_query_ids64(None, None, None, 0, 0, None, None, 0, ctypes.byref(total)) == _lib.MDRQ_EINVAL
    assert lib.mdrq_fetch_ids64(None, None, 0) == _lib.MDRQ_EINVAL
    assert lib.mdrq_last_error()


_C_PROGRAM = r"""
#include <stdio.h>
#include <stdint.h>
#include "mdrq_b200.h"
int main(void) {
    /* a C99 caller of the drop-in boundary: version, an invalid store
       (EINVAL + message), the null-store guard -- no device needed */
    mdrq_store* s = 0;
    uint64_t total = 0;
    if (mdrq_abi_version() != 1) return 2;
    if (mdrq_store_create(0, 0, 0, 0, 1, 0, 0, &s) != MDRQ_EINVAL) return 3;
    if (!mdrq_last_error() || !mdrq_last_error()[0]) return 4;
    if (mdrq_query_ids(0, 0, 0, 0, MDRQ_PATH_AUTO, 0, 0, 0, &total) != MDRQ_EINVAL) return 5;
    printf("c abi ok\n");
    return 0;
}
"""


def test_header_is_plain_c_and_links(tmp_path):
    """include/mdrq_b200.h compiles as C99 (what a cgo / FFI binding sees),
    and a C program links against libmdrq_b200.so and runs its device-free
    entry points."""
    import shutil
    import subprocess
    from paper_1801_03644_b200 import _lib
    cc = shutil.which("gcc") or shutil.which("cc")
    if not cc:
        pytest.skip("no C compiler")
    src = tmp_path / "abi.c"
    src.write_text(_C_PROGRAM)
    exe = tmp_path / "abi"
    libdir = os.path.dirname(_lib.LIB_PATH)
    r = subprocess.run([cc, "-std=c99", "-Wall", "-Werror", "-pedantic", "-I", os.path.join(ROOT, "include"),
                        str(src), "-o", str(exe), "-L", libdir, "-l:libmdrq_b200.so",
                        f"-Wl,-rpath,{libdir}"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "c abi ok" in r.stdout, (r.returncode, r.stdout, r.stderr)
