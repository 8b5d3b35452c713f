"""GPU kernel backend -- the reference's MDRQ_BACKEND plugin slot on CUDA.

Exports the names of /root/reference/pkg/src/mdrq/kernels.py:34-46 for the
hot-path kernels (``match_row``, ``scan_rows``, ``scan_column``) with the
reference's signatures and results, computed by libmdrq_b200.so on
``MDRQ_DEVICE`` (default 0).  Each call copies its inputs to HBM, so this
level exists for parity with the reference's kernel tests; the access
methods in scan.py / vafile.py keep data resident instead.

The tree kernels (kd_build, kd_search, mbr_intersect, area_enlargements,
leaf_overlap_enlargements) are out of scope.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from ._lib import check, f32p, i64p, u8p, u64p
from .store import default_device

BACKEND: str = "cuda"
MODE_SCALAR: int = _lib.MODE_SCALAR     # _kernels_cy.pyx:14
MODE_BLOCKED: int = _lib.MODE_BLOCKED   # _kernels_cy.pyx:15
LANE: int = 8                           # _kernels_cy.pyx:16


def _vec(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def match_row(row, lower, upper, mode: int) -> bool:
    """_kernels_cy.pyx:49-55: one row against one box (both modes agree)."""
    row, lo, hi = _vec(row), _vec(lower), _vec(upper)
    m = row.shape[0]
    if lo.shape[0] != m or hi.shape[0] != m:
        raise ValueError(f"bound length {lo.shape[0]} does not match m={m}")
    out = np.zeros(1, np.uint8)
    check(_lib.load().mdrq_match_rows(row.ctypes.data_as(f32p), 1, m, lo.ctypes.data_as(f32p),
                                      hi.ctypes.data_as(f32p), default_device(), out.ctypes.data_as(u8p)))
    return bool(out[0])


def match_rows(rows, lower, upper) -> np.ndarray:
    """Vectorised match_row over many rows -> bool[nrows]."""
    rows = _vec(rows)
    if rows.ndim != 2:
        raise ValueError("rows must be a 2-d matrix")
    lo, hi = _vec(lower), _vec(upper)
    n, m = rows.shape
    if lo.shape[0] != m or hi.shape[0] != m:
        raise ValueError(f"bound length {lo.shape[0]} does not match m={m}")
    out = np.zeros(max(n, 1), np.uint8)
    check(_lib.load().mdrq_match_rows(rows.ctypes.data_as(f32p), n, m, lo.ctypes.data_as(f32p),
                                      hi.ctypes.data_as(f32p), default_device(), out.ctypes.data_as(u8p)))
    return out[:n].astype(bool)


def scan_rows(values, lower, upper, mode: int):
    """_kernels_cy.pyx:58-86 -> (ascending int64 local ids, n compared, early breaks)."""
    values = np.ascontiguousarray(values, dtype=np.float32)
    if values.ndim != 2:
        raise ValueError("values must be a 2-d matrix")
    n, m = values.shape
    lo, hi = _vec(lower), _vec(upper)
    if lo.shape[0] != m or hi.shape[0] != m:
        raise ValueError(f"bound length {lo.shape[0]} does not match m={m}")
    if n == 0:
        return np.empty(0, np.int64), 0, 0
    ids = np.empty(n, np.int64)
    cnt, early = ctypes.c_uint64(0), ctypes.c_uint64(0)
    check(_lib.load().mdrq_scan_rows(values.ctypes.data_as(f32p), n, m, lo.ctypes.data_as(f32p),
                                     hi.ctypes.data_as(f32p), int(mode), default_device(),
                                     ids.ctypes.data_as(i64p), ctypes.byref(cnt), ctypes.byref(early)))
    return ids[: cnt.value].copy(), n, int(early.value)


def scan_column(col, lo, hi, mode: int = MODE_BLOCKED) -> np.ndarray:
    """_kernels_cy.pyx:89-120: packed little-endian bitmask of lo <= v <= hi."""
    col = _vec(col)
    if col.ndim != 1:
        raise ValueError("col must be 1-d")
    n = col.shape[0]
    out = np.zeros((n + 7) // 8, np.uint8)
    if n == 0:
        return out
    check(_lib.load().mdrq_scan_column(col.ctypes.data_as(f32p), n, float(np.float32(lo)),
                                       float(np.float32(hi)), default_device(), out.ctypes.data_as(u8p)))
    return out


def and_masks(masks) -> np.ndarray:
    """Bitwise AND of equal-length masks (scan.py:55-78 result)."""
    masks = [np.ascontiguousarray(mk, dtype=np.uint8) for mk in masks]
    if not masks:
        raise ValueError("no masks to merge")
    nbytes = masks[0].size
    for mk in masks:
        if mk.size != nbytes:
            raise ValueError("masks must have equal length")
    out = np.zeros(nbytes, np.uint8)
    if nbytes == 0:
        return out
    arr = (u8p * len(masks))(*[mk.ctypes.data_as(u8p) for mk in masks])
    check(_lib.load().mdrq_and_masks(arr, len(masks), nbytes, default_device(), out.ctypes.data_as(u8p)))
    return out


def mask_popcount(mask) -> int:
    """scan.py:81-82."""
    mask = np.ascontiguousarray(mask, dtype=np.uint8)
    c = ctypes.c_uint64(0)
    check(_lib.load().mdrq_mask_popcount(mask.ctypes.data_as(u8p), mask.size, default_device(),
                                         ctypes.byref(c)))
    return int(c.value)


def mask_to_ids(mask, n: int) -> np.ndarray:
    """scan.py:85-88: positions of set bits among the first n, ascending."""
    mask = np.ascontiguousarray(mask, dtype=np.uint8)
    if n > mask.size * 8:
        raise ValueError("mask shorter than n bits")
    if n == 0:
        return np.empty(0, np.int64)
    ids = np.empty(n, np.int64)
    c = ctypes.c_uint64(0)
    check(_lib.load().mdrq_mask_to_ids(mask.ctypes.data_as(u8p), n, default_device(),
                                       ids.ctypes.data_as(i64p), ctypes.byref(c)))
    return ids[: c.value].copy()


def _out_of_scope(*_a, **_k):
    raise NotImplementedError("tree-index kernels are out of scope for the GPU scan engine "
                              "(SURVEY.md section 2, rows 9-10)")


kd_build = kd_search = mbr_intersect = area_enlargements = leaf_overlap_enlargements = _out_of_scope
