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


def _pack_ids16(offsets, ids, hb0, nbuckets):
    """numpy restatement of pack.cu: the low halves and, per query, the end
    position of every 65 536-id bucket in its list."""
    nq = offsets.size - 1
    lo16 = (ids & 0xFFFF).astype(np.uint16)
    ends = np.zeros((nq, nbuckets), np.uint32)
    for q in range(nq):
        run = ids[offsets[q]:offsets[q + 1]].astype(np.int64)
        ends[q] = np.searchsorted(run, (np.arange(nbuckets, dtype=np.int64) + hb0 + 1) << 16, side="left")
    return lo16, ends


@pytest.mark.parametrize("threads", [1, 3, 16])
def test_unpack_ids16_rebuilds_the_ids(threads):
    """mdrq_unpack_ids16 (the host half of the packed device->host copy)
    needs no device: ascending id lists of ragged lengths -- empty, one id,
    lists crossing many buckets, lists inside one bucket, a shard's id base --
    packed with numpy and rebuilt by the library on 1, 3 and 16 threads."""
    from paper_1801_03644_b200 import _lib
    lib = _lib.load()
    rng = np.random.default_rng(threads)
    id_base, n = 3 * 65536 + 1234, 5_000_000
    hb0 = id_base >> 16
    nbuckets = ((id_base + n - 1) >> 16) - hb0 + 1
    runs = []
    for q in range(200):
        kind = q % 5
        cnt = [0, 1, int(rng.integers(2, 400_000)), int(rng.integers(2, 3000)), int(rng.integers(100, 60_000))][kind]
        if kind == 3:   # inside one bucket
            b = int(rng.integers(hb0 + 1, hb0 + nbuckets - 1))
            pool = np.arange(b << 16, (b + 1) << 16, dtype=np.int64)
        else:
            pool = None
        ids = (np.sort(rng.choice(pool, cnt, replace=False)) if pool is not None
               else np.sort(rng.choice(n, cnt, replace=False)) + id_base)
        runs.append(ids.astype(np.uint32))
    offsets = np.concatenate([[0], np.cumsum([r.size for r in runs])]).astype(np.uint64)
    ids = np.concatenate(runs).astype(np.uint32)
    lo16, ends = _pack_ids16(offsets.astype(np.int64), ids, hb0, nbuckets)
    out = np.full(ids.size + 8, 0xDEADBEEF, np.uint32)   # +8: nothing written past the end
    rc = lib.mdrq_unpack_ids16(lo16.ctypes.data_as(ctypes.POINTER(ctypes.c_uint16)),
                               ends.ctypes.data_as(_lib.u32p), offsets.ctypes.data_as(_lib.u64p),
                               offsets.size - 1, hb0, nbuckets, out.ctypes.data_as(_lib.u32p), threads)
    assert rc == 0
    assert np.array_equal(out[: ids.size], ids)
    assert (out[ids.size:] == 0xDEADBEEF).all()


def test_unpack_ids16_few_long_lists():
    """Threads share the ids, not the queries: three lists (one empty between
    two long ones) on 16 threads, every thread starting inside a list."""
    from paper_1801_03644_b200 import _lib
    lib = _lib.load()
    rng = np.random.default_rng(3)
    n = 40_000_000
    runs = [np.sort(rng.choice(n, 6_000_000, replace=False)).astype(np.uint32), np.empty(0, np.uint32),
            np.sort(rng.choice(n, 9_000_000, replace=False)).astype(np.uint32)]
    offsets = np.concatenate([[0], np.cumsum([r.size for r in runs])]).astype(np.uint64)
    ids = np.concatenate(runs)
    nbuckets = ((n - 1) >> 16) + 1
    lo16, ends = _pack_ids16(offsets.astype(np.int64), ids, 0, nbuckets)
    out = np.zeros(ids.size, np.uint32)
    rc = lib.mdrq_unpack_ids16(lo16.ctypes.data_as(ctypes.POINTER(ctypes.c_uint16)), ends.ctypes.data_as(_lib.u32p),
                               offsets.ctypes.data_as(_lib.u64p), 3, 0, nbuckets, out.ctypes.data_as(_lib.u32p), 16)
    assert rc == 0 and np.array_equal(out, ids)
