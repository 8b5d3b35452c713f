"""ctypes binding of libmdrq_b200.so (include/mdrq_b200.h).

The shared library is the product's only compute path.  Loading it never
needs a GPU (cudart is linked statically and the driver is opened lazily),
but every compute entry point fails loudly -- RuntimeError / ValueError --
when no CUDA device is present.  There is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
# MDRQ_LIB=checked loads the build with device-side bounds checks
# (build.py --checked, common.cuh MDRQ_CHECKS) -- for tests
# (any other MDRQ_LIB=<name>: an experiment build, build.py --variant <name>)
LIB_PATH = os.path.join(PKG, f"libmdrq_b200_{os.environ['MDRQ_LIB']}.so" if os.environ.get("MDRQ_LIB")
                        else "libmdrq_b200.so")

MDRQ_OK = 0
MDRQ_EINVAL = -1
MDRQ_ECUDA = -2
MDRQ_ENOMEM = -3
MDRQ_ETRUNC = -4
MDRQ_ENODEV = -5

LAYOUT_COLUMNAR = 1
LAYOUT_ROWWISE = 2
LAYOUT_VAFILE = 4

PATH_AUTO = 0
PATH_COLUMNAR = 1
PATH_ROWWISE = 2
PATH_VAFILE = 3
PATH_COLUMNAR_BATCH = 4
PATH_VAFILE_BATCH = 5

PATHS = {
    "auto": PATH_AUTO,
    "columnar": PATH_COLUMNAR,
    "rowwise": PATH_ROWWISE,
    "vafile": PATH_VAFILE,
    "columnar_batch": PATH_COLUMNAR_BATCH,
    "vafile_batch": PATH_VAFILE_BATCH,
}

MODE_SCALAR = 0
MODE_BLOCKED = 1

#: every symbol include/mdrq_b200.h declares (checked by tests/test_abi.py)
EXPORTED = (
    "mdrq_last_error", "mdrq_abi_version", "mdrq_check_flags", "mdrq_device_count", "mdrq_measure_read_bw", "mdrq_copy_segments",
    "mdrq_copy_segments_dma",
    "mdrq_match_rows", "mdrq_scan_rows", "mdrq_scan_column", "mdrq_and_masks",
    "mdrq_mask_popcount", "mdrq_mask_to_ids",
    "mdrq_store_create", "mdrq_store_destroy", "mdrq_store_get_info",
    "mdrq_store_va_boundaries", "mdrq_store_bounds",
    "mdrq_query_count", "mdrq_query_ids", "mdrq_fetch_ids", "mdrq_query_ids64", "mdrq_fetch_ids64", "mdrq_query_ids_stream", "mdrq_unpack_ids16", "mdrq_stream_info", "mdrq_query_stats",
    "mdrq_batch_prepare", "mdrq_batch_destroy", "mdrq_batch_count_async",
    "mdrq_batch_ids_async", "mdrq_batch_reserve", "mdrq_result_device",
    "mdrq_batch_launches", "mdrq_batch_profile", "mdrq_batch_info",
)


class StoreInfo(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_uint64),
        ("m", ctypes.c_uint32),
        ("layouts", ctypes.c_uint32),
        ("va_bits", ctypes.c_uint32),
        ("device", ctypes.c_int32),
        ("n_pad", ctypes.c_uint64),
        ("device_bytes", ctypes.c_uint64),
    ]


class SearchStatsC(ctypes.Structure):
    _fields_ = [
        ("objects_compared", ctypes.c_uint64),
        ("nodes_visited", ctypes.c_uint64),
        ("columns_scanned", ctypes.c_uint64),
        ("early_breaks", ctypes.c_uint64),
        ("and_chunks", ctypes.c_uint64),
        ("bytes_loaded", ctypes.c_uint64),
    ]


_f32p = ctypes.POINTER(ctypes.c_float)
_u8p = ctypes.POINTER(ctypes.c_uint8)
_u32p = ctypes.POINTER(ctypes.c_uint32)
_u64p = ctypes.POINTER(ctypes.c_uint64)
_i64p = ctypes.POINTER(ctypes.c_int64)
_vp = ctypes.c_void_p
_u32 = ctypes.c_uint32
_u64 = ctypes.c_uint64
_int = ctypes.c_int

_SIGS = {
    "mdrq_last_error": (ctypes.c_char_p, []),
    "mdrq_copy_segments_dma": (_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64),
                                      ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64),
                                      ctypes.c_uint64, ctypes.c_void_p]),
    "mdrq_abi_version": (_int, []),
    "mdrq_unpack_ids16": (_int, [ctypes.POINTER(ctypes.c_uint16), _u32p, _u64p, _u32, _u32, _u32, _u32p, _int]),
    "mdrq_stream_info": (_int, [_vp, _u64p]),
    "mdrq_check_flags": (_int, [ctypes.POINTER(ctypes.c_uint32)]),
    "mdrq_device_count": (_int, [ctypes.POINTER(_int)]),
    "mdrq_measure_read_bw": (_int, [_int, _u64, _int, ctypes.POINTER(ctypes.c_double)]),
    "mdrq_copy_segments": (_int, [_vp, _vp, _vp, _vp, _vp, _u64, _vp]),
    "mdrq_match_rows": (_int, [_f32p, _u64, _u32, _f32p, _f32p, _int, _u8p]),
    "mdrq_scan_rows": (_int, [_f32p, _u64, _u32, _f32p, _f32p, _int, _int, _i64p, _u64p, _u64p]),
    "mdrq_scan_column": (_int, [_f32p, _u64, ctypes.c_float, ctypes.c_float, _int, _u8p]),
    "mdrq_and_masks": (_int, [ctypes.POINTER(_u8p), _u32, _u64, _int, _u8p]),
    "mdrq_mask_popcount": (_int, [_u8p, _u64, _int, _u64p]),
    "mdrq_mask_to_ids": (_int, [_u8p, _u64, _int, _i64p, _u64p]),
    "mdrq_store_create": (_int, [_f32p, _u64, _u32, _int, _u32, _u32, _u64, ctypes.POINTER(_vp)]),
    "mdrq_store_destroy": (_int, [_vp]),
    "mdrq_store_get_info": (_int, [_vp, ctypes.POINTER(StoreInfo)]),
    "mdrq_store_va_boundaries": (_int, [_vp, _f32p]),
    "mdrq_store_bounds": (_int, [_vp, _f32p]),
    "mdrq_query_count": (_int, [_vp, _f32p, _f32p, _u32, _u32, _u64p]),
    "mdrq_query_ids": (_int, [_vp, _f32p, _f32p, _u32, _u32, _u64p, _u32p, _u64, _u64p]),
    "mdrq_fetch_ids": (_int, [_vp, _u32p, _u64]),
    "mdrq_query_ids64": (_int, [_vp, _f32p, _f32p, _u32, _u32, _u64p, _i64p, _u64, _u64p]),
    "mdrq_fetch_ids64": (_int, [_vp, _i64p, _u64]),
    "mdrq_query_ids_stream": (_int, [_vp, _f32p, _f32p, _u32p, _u32, _u32, ctypes.POINTER(_u64p),
                                     ctypes.POINTER(_u32p), _u64p, _u64p, _u64p]),
    "mdrq_query_stats": (_int, [_vp, _int, ctypes.POINTER(SearchStatsC), _u32]),
    "mdrq_batch_prepare": (_int, [_vp, _f32p, _f32p, _u32, _u32, ctypes.POINTER(_vp)]),
    "mdrq_batch_destroy": (_int, [_vp]),
    "mdrq_batch_count_async": (_int, [_vp, _vp, _vp, _vp]),
    "mdrq_batch_ids_async": (_int, [_vp, _vp, _vp]),
    "mdrq_batch_reserve": (_int, [_vp, _vp, _u64p]),
    "mdrq_result_device": (_int, [_vp, _u64p, _u64p, _u64p]),
    "mdrq_batch_launches": (_int, [_vp, _int, _u32p]),
    "mdrq_batch_profile": (_int, [_vp, _vp, _int, _vp, ctypes.POINTER(ctypes.c_double), _u32p]),
    "mdrq_batch_info": (_int, [_vp, _u32p]),
}

_lock = threading.Lock()
_LIB = None


class MdrqError(RuntimeError):
    """CUDA-side failure of the engine (no CPU fallback exists)."""


def load():
    """Load libmdrq_b200.so; raises ImportError if it has not been built."""
    global _LIB
    if _LIB is not None:
        return _LIB
    with _lock:
        if _LIB is not None:
            return _LIB
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_1801_03644_b200.build` "
                "(the GPU engine has no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = lib
    return _LIB


def last_error() -> str:
    return load().mdrq_last_error().decode("utf-8", "replace")


def check(rc: int) -> int:
    if rc == MDRQ_OK:
        return rc
    msg = last_error()
    if rc == MDRQ_EINVAL:
        raise ValueError(msg)
    if rc == MDRQ_ENOMEM:
        raise MemoryError(msg)
    raise MdrqError(f"libmdrq_b200 error {rc}: {msg}")


def device_count() -> int:
    c = ctypes.c_int(0)
    check(load().mdrq_device_count(ctypes.byref(c)))
    return int(c.value)


def ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


f32p, u8p, u32p, u64p, i64p = _f32p, _u8p, _u32p, _u64p, _i64p
