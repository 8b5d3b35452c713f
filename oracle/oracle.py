"""Oracle implementation (see oracle/__init__.py: test infrastructure only)."""

from __future__ import annotations

import ctypes
import importlib.util
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

import numpy as np

__all__ = [
    "HERE", "lib", "build_oracle",
    "match_code", "match_row", "scan_rows", "scan_column",
    "and_masks", "mask_popcount", "mask_to_ids",
    "count_batch", "ids_batch", "hash_batch", "id_hash", "set_hash", "va_code", "va_encode",
    "brute_ids", "brute_mask", "packbits_mask", "chunk_spans",
    "and_masks_chunked", "np_mask_to_ids",
    "load_reference_kernels", "reference_kind", "ReferenceHorizontalScan",
    "make_layout_ids",
]

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

_f32p = ctypes.POINTER(ctypes.c_float)
_i64p = ctypes.POINTER(ctypes.c_int64)
_u8p = ctypes.POINTER(ctypes.c_uint8)


def build_oracle(ref: bool = False) -> None:
    """Compile the C restatement (and, if asked and present, the reference)."""
    targets = ["oracle"] + (["ref"] if ref else [])
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


def lib():
    global _LIB
    if _LIB is not None:
        return _LIB
    path = os.path.join(HERE, "libmdrq_oracle.so")
    if not os.path.exists(path):
        build_oracle()
    L = ctypes.CDLL(path)
    L.oracle_match_code.restype = ctypes.c_int
    L.oracle_match_code.argtypes = [_f32p, _f32p, _f32p, ctypes.c_int64, ctypes.c_int]
    L.oracle_match_row.restype = ctypes.c_int
    L.oracle_match_row.argtypes = [_f32p, _f32p, _f32p, ctypes.c_int64, ctypes.c_int]
    L.oracle_scan_rows.restype = ctypes.c_int64
    L.oracle_scan_rows.argtypes = [_f32p, ctypes.c_int64, ctypes.c_int64, _f32p, _f32p,
                                   ctypes.c_int, _i64p, _i64p]
    L.oracle_scan_column.restype = None
    L.oracle_scan_column.argtypes = [_f32p, ctypes.c_int64, ctypes.c_float, ctypes.c_float, _u8p]
    L.oracle_and_masks.restype = None
    L.oracle_and_masks.argtypes = [ctypes.POINTER(_u8p), ctypes.c_int64, ctypes.c_int64, _u8p]
    L.oracle_mask_popcount.restype = ctypes.c_int64
    L.oracle_mask_popcount.argtypes = [_u8p, ctypes.c_int64]
    L.oracle_mask_to_ids.restype = ctypes.c_int64
    L.oracle_mask_to_ids.argtypes = [_u8p, ctypes.c_int64, _i64p]
    L.oracle_count_batch.restype = None
    L.oracle_count_batch.argtypes = [_f32p, ctypes.c_int64, ctypes.c_int64, _f32p, _f32p,
                                     ctypes.c_int64, _i64p, ctypes.c_int]
    L.oracle_ids_batch.restype = None
    L.oracle_ids_batch.argtypes = [_f32p, ctypes.c_int64, ctypes.c_int64, _f32p, _f32p,
                                   ctypes.c_int64, _i64p, _i64p, ctypes.c_int]
    L.oracle_va_code.restype = ctypes.c_int32
    L.oracle_va_code.argtypes = [_f32p, ctypes.c_int32, ctypes.c_float]
    L.oracle_va_encode.restype = None
    L.oracle_va_encode.argtypes = [_f32p, ctypes.c_int64, _f32p, ctypes.c_int32, _u8p]
    L.oracle_has_openmp.restype = ctypes.c_int
    L.oracle_hash_batch.restype = ctypes.c_int
    L.oracle_hash_batch.argtypes = [_f32p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, _f32p, _f32p,
                                    ctypes.c_int64, _i64p, ctypes.POINTER(ctypes.c_uint64), ctypes.c_int]
    L.oracle_id_hash.restype = ctypes.c_uint64
    L.oracle_id_hash.argtypes = [ctypes.c_uint64]
    _LIB = L
    return L


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _p(a, t):
    return a.ctypes.data_as(t)


# -- C restatement wrappers ---------------------------------------------------

def match_code(row, lower, upper, mode: int) -> int:
    """_kernels_cy.pyx:23-46: 1 match, 0 fail at last dim, -1 early break."""
    row, lo, hi = _f32(row), _f32(lower), _f32(upper)
    return lib().oracle_match_code(_p(row, _f32p), _p(lo, _f32p), _p(hi, _f32p), row.size, mode)


def match_row(row, lower, upper, mode: int) -> bool:
    """_kernels_cy.pyx:49-55."""
    row, lo, hi = _f32(row), _f32(lower), _f32(upper)
    if lo.shape[0] != row.shape[0] or hi.shape[0] != row.shape[0]:
        raise ValueError(f"bound length {lo.shape[0]} does not match m={row.shape[0]}")
    return bool(lib().oracle_match_row(_p(row, _f32p), _p(lo, _f32p), _p(hi, _f32p),
                                       row.size, mode))


def scan_rows(values, lower, upper, mode: int):
    """_kernels_cy.pyx:58-86 -> (ids int64 ascending, n, early breaks)."""
    values = _f32(values)
    n, m = values.shape
    lo, hi = _f32(lower), _f32(upper)
    if lo.shape[0] != m or hi.shape[0] != m:
        raise ValueError(f"bound length {lo.shape[0]} does not match m={m}")
    out = np.empty(max(n, 1), dtype=np.int64)
    early = ctypes.c_int64(0)
    cnt = lib().oracle_scan_rows(_p(values, _f32p), n, m, _p(lo, _f32p), _p(hi, _f32p),
                                 mode, _p(out, _i64p), ctypes.byref(early))
    return out[:cnt].copy(), n, int(early.value)


def scan_column(col, lo: float, hi: float) -> np.ndarray:
    """_kernels_cy.pyx:89-120 (mode-independent result)."""
    col = _f32(col)
    out = np.empty((col.size + 7) // 8, dtype=np.uint8)
    lib().oracle_scan_column(_p(col, _f32p), col.size, float(np.float32(lo)),
                             float(np.float32(hi)), _p(out, _u8p))
    return out


def and_masks(masks) -> np.ndarray:
    masks = [np.ascontiguousarray(mk, dtype=np.uint8) for mk in masks]
    nbytes = masks[0].size
    arr = (_u8p * len(masks))(*[_p(mk, _u8p) for mk in masks])
    out = np.empty(nbytes, dtype=np.uint8)
    lib().oracle_and_masks(arr, len(masks), nbytes, _p(out, _u8p))
    return out


def mask_popcount(mask) -> int:
    mask = np.ascontiguousarray(mask, dtype=np.uint8)
    return int(lib().oracle_mask_popcount(_p(mask, _u8p), mask.size))


def mask_to_ids(mask, n: int) -> np.ndarray:
    mask = np.ascontiguousarray(mask, dtype=np.uint8)
    out = np.empty(max(n, 1), dtype=np.int64)
    c = lib().oracle_mask_to_ids(_p(mask, _u8p), n, _p(out, _i64p))
    return out[:c].copy()


def count_batch(values, lower, upper, threads: int = 0) -> np.ndarray:
    """SequentialScan (scan.py:103-111) over a query batch: counts int64[nq]."""
    values = _f32(values)
    n, m = values.shape
    lo = _f32(lower).reshape(-1, m)
    hi = _f32(upper).reshape(-1, m)
    nq = lo.shape[0]
    counts = np.zeros(nq, dtype=np.int64)
    if nq:
        lib().oracle_count_batch(_p(values, _f32p), n, m, _p(lo, _f32p), _p(hi, _f32p),
                                 nq, _p(counts, _i64p), threads)
    return counts


def ids_batch(values, lower, upper, threads: int = 0, counts=None):
    """SequentialScan over a batch -> (offsets int64[nq+1], ids int64[total])."""
    values = _f32(values)
    n, m = values.shape
    lo = _f32(lower).reshape(-1, m)
    hi = _f32(upper).reshape(-1, m)
    nq = lo.shape[0]
    if counts is None:
        counts = count_batch(values, lo, hi, threads)
    offsets = np.zeros(nq + 1, dtype=np.int64)
    np.cumsum(counts, out=offsets[1:])
    ids = np.empty(max(int(offsets[-1]), 1), dtype=np.int64)
    if nq:
        lib().oracle_ids_batch(_p(values, _f32p), n, m, _p(lo, _f32p), _p(hi, _f32p), nq,
                               _p(offsets, _i64p), _p(ids, _i64p), threads)
    return offsets, ids[:offsets[-1]]


def hash_batch(values, lower, upper, id0: int = 0, counts=None, hashes=None, threads: int = 0):
    """SequentialScan (scan.py:103-111) over a batch reduced to per-query
    (count, set hash): hashes[q] = sum of id_hash(id) over the matching ids,
    mod 2**64 (mdrq_oracle.c oracle_hash_batch).  ``values`` are rows
    id0 .. id0+n-1; results are accumulated into ``counts`` / ``hashes`` when
    given, so a table can be streamed through in row chunks."""
    values = _f32(values)
    n, m = values.shape
    lo = _f32(lower).reshape(-1, m)
    hi = _f32(upper).reshape(-1, m)
    nq = lo.shape[0]
    if counts is None:
        counts = np.zeros(nq, dtype=np.int64)
    if hashes is None:
        hashes = np.zeros(nq, dtype=np.uint64)
    assert counts.dtype == np.int64 and hashes.dtype == np.uint64 and counts.flags.c_contiguous
    rc = lib().oracle_hash_batch(_p(values, _f32p), n, m, int(id0), _p(lo, _f32p), _p(hi, _f32p), nq,
                                 _p(counts, _i64p), hashes.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
                                 threads)
    if rc != 0:
        raise ValueError("NaN values are rejected at ingestion")
    return counts, hashes


_MIX = (np.uint64(0x9E3779B97F4A7C15), np.uint64(0xBF58476D1CE4E5B9), np.uint64(0x94D049BB133111EB))


def id_hash(ids) -> np.ndarray:
    """splitmix64 finalizer of every id (numpy, uint64 wraparound); the C
    oracle's oracle_mix64."""
    z = np.asarray(ids).astype(np.uint64) + _MIX[0]
    z = (z ^ (z >> np.uint64(30))) * _MIX[1]
    z = (z ^ (z >> np.uint64(27))) * _MIX[2]
    return z ^ (z >> np.uint64(31))


def set_hash(offsets, ids) -> np.ndarray:
    """Per-query set hash of an (offsets, ids) result, as hash_batch
    computes it: the sum mod 2**64 of id_hash over each query's ids."""
    offsets = np.asarray(offsets, dtype=np.int64)
    h = id_hash(ids)
    c = np.zeros(h.size + 1, dtype=np.uint64)
    np.cumsum(h, out=c[1:])
    return c[offsets[1:]] - c[offsets[:-1]]


def va_code(boundaries, v: float) -> int:
    b = _f32(boundaries)
    return int(lib().oracle_va_code(_p(b, _f32p), b.size, float(np.float32(v))))


def va_encode(col, boundaries) -> np.ndarray:
    col, b = _f32(col), _f32(boundaries)
    out = np.empty(col.size, dtype=np.uint8)
    lib().oracle_va_encode(_p(col, _f32p), col.size, _p(b, _f32p), b.size, _p(out, _u8p))
    return out


# -- numpy restatements -------------------------------------------------------

def brute_mask(values, lower, upper) -> np.ndarray:
    """pkg/tests/test_scan.py:22-28 as a bool mask (plain numpy containment)."""
    values = _f32(values)
    lo, hi = _f32(lower), _f32(upper)
    ok = np.ones(values.shape[0], dtype=bool)
    for j in range(values.shape[1]):
        col = values[:, j]
        ok &= (col >= lo[j]) & (col <= hi[j])
    return ok


def brute_ids(values, lower, upper) -> np.ndarray:
    """pkg/tests/test_scan.py:22-28: the reference suite's independent oracle."""
    return np.flatnonzero(brute_mask(values, lower, upper)).astype(np.int64)


def packbits_mask(col, lo, hi) -> np.ndarray:
    """pkg/tests/test_kernels.py:109 expected scan_column mask."""
    col = _f32(col)
    return np.packbits((col >= np.float32(lo)) & (col <= np.float32(hi)), bitorder="little")


def chunk_spans(nbytes: int, t: int):
    """scan.py:43-52."""
    if t < 1:
        raise ValueError("chunk count must be at least 1")
    size = -(-nbytes // t)
    spans = []
    for i in range(t):
        start = min(i * size, nbytes)
        spans.append((start, min(start + size, nbytes)))
    return spans


def and_masks_chunked(masks, t: int) -> np.ndarray:
    """scan.py:55-78 without the pool."""
    masks = list(masks)
    if not masks:
        raise ValueError("no masks to merge")
    out = np.empty(masks[0].shape[0], dtype=np.uint8)
    for start, end in chunk_spans(out.size, t):
        if start == end:
            continue
        acc = out[start:end]
        acc[:] = masks[0][start:end]
        for mk in masks[1:]:
            np.bitwise_and(acc, mk[start:end], out=acc)
    return out


def np_mask_to_ids(mask, n: int) -> np.ndarray:
    """scan.py:85-88."""
    return np.flatnonzero(np.unpackbits(mask, count=n, bitorder="little")).astype(np.int64)


# -- the reference's own compiled kernels (oracle/_ref) -----------------------

def _cpu_flags() -> set:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("flags"):
                    return set(line.split(":", 1)[1].split())
    except OSError:
        pass
    return set()


_REF = None
_REF_KIND = None


def load_reference_kernels():
    """Import the reference's ``_kernels_cy`` built by oracle/Makefile, or None.

    Picks the x86-64-v3 build when the host has AVX2/FMA/BMI2, else the
    generic build.  Returns the module (BACKEND == "compiled").
    """
    global _REF, _REF_KIND
    if _REF is not None:
        return _REF
    flags = _cpu_flags()
    variants = (["v3"] if {"avx2", "fma", "bmi2"} <= flags else []) + ["generic"]
    suffix = __import__("sysconfig").get_config_var("EXT_SUFFIX")
    for v in variants:
        path = os.path.join(HERE, "_ref", v, "_kernels_cy" + suffix)
        if not os.path.exists(path):
            continue
        spec = importlib.util.spec_from_file_location("_kernels_cy", path)
        mod = importlib.util.module_from_spec(spec)
        try:
            spec.loader.exec_module(mod)
        except ImportError:
            continue
        sys.modules.setdefault("_mdrq_ref_kernels_cy", mod)
        _REF, _REF_KIND = mod, f"reference _kernels_cy ({v} build)"
        return mod
    return None


def reference_kind() -> str | None:
    load_reference_kernels()
    return _REF_KIND


def make_layout_ids(n: int, p: int, seed: int):
    """parallel.py:98-118 (make_layout): seeded permutation split into p runs,
    the first n mod p partitions one larger."""
    if p < 1:
        raise ValueError("partition count must be at least 1")
    perm = np.random.default_rng(seed).permutation(n).astype(np.int64)
    base, extra = divmod(n, p)
    parts, start = [], 0
    for q in range(p):
        size = base + (1 if q < extra else 0)
        parts.append(perm[start:start + size])
        start += size
    return parts


class ReferenceHorizontalScan:
    """The reference's HorizontalScan (scan.py:117-164) driven by the
    reference's own compiled ``scan_rows`` (``_ref``) -- or, when that build
    is absent, by the C restatement (``kind == "port"``).

    Random row partitions are gathered into contiguous blocks (scan.py:129-132),
    each query fans out one ``scan_rows`` task per block over a thread pool
    (the GIL is released inside the kernel, _kernels_cy.pyx:78), local ids are
    mapped to global ids (scan.py:149) and merged by concatenate + sort
    (scan.py:160).
    """

    def __init__(self, values, threads: int, seed: int = 0, mode: int = 0):
        values = _f32(values)
        self.n, self.m = values.shape
        self.mode = mode
        self.threads = max(1, int(threads))
        ref = load_reference_kernels()
        self.kind = "reference" if ref is not None else "port"
        self._scan = ref.scan_rows if ref is not None else scan_rows
        parts = make_layout_ids(self.n, self.threads, seed)
        self._parts = [(np.ascontiguousarray(values[ids]), ids.copy()) for ids in parts]
        self._pool = ThreadPoolExecutor(max_workers=self.threads) if self.threads > 1 else None

    def search(self, lower, upper) -> np.ndarray:
        lo, hi = _f32(lower), _f32(upper)

        def task(block, ids):
            local, _, _ = self._scan(block, lo, hi, self.mode)
            return ids[local]

        if self._pool is None:
            chunks = [task(b, i) for b, i in self._parts]
        else:
            futs = [self._pool.submit(task, b, i) for b, i in self._parts]
            chunks = [f.result() for f in futs]
        chunks = [c for c in chunks if c.size]
        return np.sort(np.concatenate(chunks)) if chunks else np.empty(0, np.int64)

    def close(self):
        if self._pool is not None:
            self._pool.shutdown(wait=True)
            self._pool = None
