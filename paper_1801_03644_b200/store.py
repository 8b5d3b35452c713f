"""Device-resident MDRQ store: the Python handle of an ``mdrq_store``.

One store holds one row shard of a dataset in HBM in up to three layouts
(DESIGN.md "Data layout"):

* columnar  -- m float32 columns of n_pad entries (NaN padded);
* row-wise  -- the row-major float32 matrix, padded to whole row tiles;
* VA-file   -- one byte plane of quantile-grid codes per dimension, plus
  the columns for exact refinement.

Queries go in as float32 ``lower``/``upper`` matrices [nq, m] with the
reference's +-inf sentinels; ids come back ascending (uint32 on the device,
widened to int64 only where the reference API demands it).
"""

from __future__ import annotations

import ctypes
import os
import threading
import weakref

import numpy as np

from . import _lib
from ._lib import check, f32p, i64p, u32p, u64p

DEFAULT_VA_BITS = 8


def default_device() -> int:
    env = os.environ.get("MDRQ_DEVICE")
    if env:
        return int(env)
    try:
        import torch
        if torch.cuda.is_available():
            return torch.cuda.current_device()
    except Exception:  # pragma: no cover - torch is optional plumbing
        pass
    return 0


def _bounds(lower, upper, m: int):
    lo = np.ascontiguousarray(lower, dtype=np.float32).reshape(-1, m)
    hi = np.ascontiguousarray(upper, dtype=np.float32).reshape(-1, m)
    if lo.shape != hi.shape:
        raise ValueError("lower and upper must have the same shape")
    return lo, hi


class DeviceStore:
    """Owns one ``mdrq_store`` (device arrays + result pool)."""

    def __init__(self, values, *, layouts: int = _lib.LAYOUT_COLUMNAR, va_bits: int = DEFAULT_VA_BITS,
                 device: int | None = None, id_base: int = 0):
        lib = _lib.load()
        values = np.ascontiguousarray(values, dtype=np.float32)
        if values.ndim != 2:
            raise ValueError(f"expected a 2-d value matrix, got shape {values.shape}")
        self.n, self.m = (int(x) for x in values.shape)
        self.device = default_device() if device is None else int(device)
        self.id_base = int(id_base)
        if not layouts & _lib.LAYOUT_VAFILE:
            va_bits = 0
        handle = ctypes.c_void_p()
        check(lib.mdrq_store_create(values.ctypes.data_as(f32p), self.n, self.m, self.device,
                                    layouts, va_bits, self.id_base, ctypes.byref(handle)))
        self._h = handle
        # one store is not re-entrant across paired C calls (query + fetch,
        # ids + stats share the store's cached result): one lock per store
        self._lock = threading.RLock()
        self._batches = weakref.WeakSet()
        info = _lib.StoreInfo()
        check(lib.mdrq_store_get_info(self._h, ctypes.byref(info)))
        self.layouts = int(info.layouts)
        self.va_bits = int(info.va_bits)
        self.n_pad = int(info.n_pad)

    @classmethod
    def from_file(cls, path, *, shard: tuple[int, int] | None = None, layouts: int = _lib.LAYOUT_COLUMNAR,
                  va_bits: int = DEFAULT_VA_BITS, device: int | None = None) -> "DeviceStore":
        """Stream a dataset file in the reference's binary format (magic
        'MDRQ' v1, core.py:295-320) into a device store.  With
        ``shard=(rank, world)`` only this rank's contiguous row range is
        read (memory-mapped, so a 20 GB file never sits in host RAM twice)
        and the store's ids start at the shard's first row (SURVEY.md 8f
        item 2)."""
        import os

        from .core import read_header
        from .parallel import shard_range
        n, m, off = read_header(path)
        payload = os.path.getsize(path) - off
        if payload != n * m * 4:
            raise ValueError(f"{path}: payload is {payload} bytes, expected {n * m * 4} for n={n} m={m}")
        start, stop = (0, n) if shard is None else shard_range(n, shard[1], shard[0])
        if n == 0:
            rows = np.empty((0, m), np.float32)
        else:
            mm = np.memmap(path, dtype="<f4", mode="r", offset=off, shape=(n, m))
            rows = np.asarray(mm[start:stop], dtype=np.float32)
        for s in range(0, rows.shape[0], 1 << 22):
            if np.isnan(rows[s:s + (1 << 22)]).any():
                raise ValueError("NaN values are rejected at ingestion")
        return cls(rows, layouts=layouts, va_bits=va_bits, device=device, id_base=start)

    # -- lifecycle -----------------------------------------------------------
    @property
    def handle(self):
        if self._h is None:
            raise ValueError("store is closed")
        return self._h

    def close(self) -> None:
        for b in list(getattr(self, "_batches", ())):
            b.close()   # prepared batches first (the C side also detaches them)
        h, self._h = getattr(self, "_h", None), None
        if h:
            _lib.load().mdrq_store_destroy(h)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- info ----------------------------------------------------------------
    def info(self) -> dict:
        info = _lib.StoreInfo()
        check(_lib.load().mdrq_store_get_info(self.handle, ctypes.byref(info)))
        return {f: getattr(info, f) for f, _ in info._fields_}

    def va_boundaries(self) -> np.ndarray:
        nb = (1 << self.va_bits) - 1
        out = np.empty((self.m, nb), np.float32)
        check(_lib.load().mdrq_store_va_boundaries(self.handle, out.ctypes.data_as(f32p)))
        return out

    def bounds(self) -> np.ndarray:
        out = np.empty((self.m, 2), np.float32)
        check(_lib.load().mdrq_store_bounds(self.handle, out.ctypes.data_as(f32p)))
        return out

    # -- one-shot queries ---------------------------------------------------
    def count(self, lower, upper, path: str | int = "auto") -> np.ndarray:
        lo, hi = _bounds(lower, upper, self.m)
        nq = lo.shape[0]
        counts = np.zeros(nq, np.uint64)
        with self._lock:
            check(_lib.load().mdrq_query_count(self.handle, lo.ctypes.data_as(f32p), hi.ctypes.data_as(f32p),
                                               nq, _path(path), counts.ctypes.data_as(u64p)))
        return counts.astype(np.int64)

    def ids(self, lower, upper, path: str | int = "auto", out: np.ndarray | None = None):
        """-> (offsets int64[nq+1], ids uint32[total]) ascending per query.

        ``out`` may be a caller-owned (e.g. pinned) uint32 buffer; the ids are
        written into its prefix and that view is returned.
        """
        lib = _lib.load()
        lo, hi = _bounds(lower, upper, self.m)
        nq = lo.shape[0]
        offsets = np.zeros(nq + 1, np.uint64)
        total = ctypes.c_uint64(0)
        buf = out if out is not None else np.empty(max(1, _guess(self.n, nq)), np.uint32)
        with self._lock:
            rc = lib.mdrq_query_ids(self.handle, lo.ctypes.data_as(f32p), hi.ctypes.data_as(f32p), nq,
                                    _path(path), offsets.ctypes.data_as(u64p), buf.ctypes.data_as(u32p),
                                    buf.size, ctypes.byref(total))
            if rc == _lib.MDRQ_ETRUNC:
                if out is not None:
                    raise ValueError(f"ids buffer holds {out.size} ids, the batch produced {total.value}")
                buf = np.empty(int(total.value), np.uint32)
                check(lib.mdrq_fetch_ids(self.handle, buf.ctypes.data_as(u32p), buf.size))
            else:
                check(rc)
        return offsets.astype(np.int64), buf[: int(total.value)]

    def ids64(self, lower, upper, path: str | int = "auto"):
        """-> (offsets int64[nq+1], ids int64[total]): ``ids`` with the ids
        widened on the host into an exactly sized array -- the dtype of the
        reference's ResultSet (core.py:185).  Two C calls: the query (which
        reports the total and keeps a small result in pinned host memory),
        then the widening copy into the fresh array."""
        lib = _lib.load()
        lo, hi = _bounds(lower, upper, self.m)
        nq = lo.shape[0]
        offsets = np.zeros(nq + 1, np.uint64)
        total = ctypes.c_uint64(0)
        with self._lock:
            rc = lib.mdrq_query_ids64(self.handle, lo.ctypes.data_as(f32p), hi.ctypes.data_as(f32p), nq,
                                      _path(path), offsets.ctypes.data_as(u64p), None, 0, ctypes.byref(total))
            ids = np.empty(int(total.value), np.int64)
            if rc == _lib.MDRQ_ETRUNC:
                check(lib.mdrq_fetch_ids64(self.handle, ids.ctypes.data_as(i64p), ids.size))
            else:
                check(rc)
        return offsets.view(np.int64), ids

    def ids64_with_stats(self, lower, upper, path: str | int = "auto", mode: int = _lib.MODE_SCALAR):
        """ids64 and the pass's per-query counters, under one hold of the
        store's lock (no other thread's call can replace the cached batch
        between the two)."""
        with self._lock:
            offs, ids = self.ids64(lower, upper, path)
            return offs, ids, self.stats(offs.size - 1, mode)

    def ids_stream(self, batches, path: str | int = "auto", outs=None, info: dict | None = None):
        """Pipelined ids for a sequence of query batches ``[(lower, upper),
        ...]`` -> list of ``(offsets int64[nq+1], ids uint32[total])``, one per
        batch, each exactly what :meth:`ids` returns for it.  Batch k's
        device->host copies overlap batch k+1's scan (mdrq_query_ids_stream).

        ``outs`` optionally gives one caller-owned (e.g. pinned) uint32 buffer
        per batch; a batch that does not fit its buffer raises ValueError.
        ``info``, when a dict, receives ``h2d_bytes`` (descriptor bytes
        uploaded), ``totals``, ``d2h_bytes`` and ``packed_batches`` (large
        results cross PCIe as 16-bit low halves + per-query bucket ends and
        are rebuilt on the host's threads, mdrq_unpack_ids16).
        """
        lib = _lib.load()
        pairs = [_bounds(lo, hi, self.m) for lo, hi in batches]
        nb = len(pairs)
        if nb == 0:
            return []
        if outs is not None and len(outs) != nb:
            raise ValueError(f"{len(outs)} output buffers for {nb} batches")
        nqs = np.array([p[0].shape[0] for p in pairs], np.uint32)
        lo_all = np.ascontiguousarray(np.concatenate([p[0] for p in pairs]), np.float32)
        hi_all = np.ascontiguousarray(np.concatenate([p[1] for p in pairs]), np.float32)
        offs = [np.zeros(int(q) + 1, np.uint64) for q in nqs]
        bufs = list(outs) if outs is not None else [np.empty(max(1, _guess(self.n, int(q))), np.uint32)
                                                    for q in nqs]
        caps = np.array([b.size for b in bufs], np.uint64)
        totals = np.zeros(nb, np.uint64)
        h2d = ctypes.c_uint64(0)
        offs_p = (u64p * nb)(*[o.ctypes.data_as(u64p) for o in offs])
        ids_p = (u32p * nb)(*[b.ctypes.data_as(u32p) for b in bufs])
        with self._lock:
            rc = lib.mdrq_query_ids_stream(self.handle, lo_all.ctypes.data_as(f32p), hi_all.ctypes.data_as(f32p),
                                           nqs.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)), nb,
                                           _path(path), offs_p, ids_p, caps.ctypes.data_as(u64p),
                                           totals.ctypes.data_as(u64p), ctypes.byref(h2d))
        if rc != _lib.MDRQ_ETRUNC:
            check(rc)
        out = []
        for k in range(nb):
            if totals[k] > caps[k]:
                if outs is not None:
                    raise ValueError(f"ids buffer {k} holds {caps[k]} ids, the batch produced {totals[k]}")
                out.append(self.ids(pairs[k][0], pairs[k][1], path))   # rare: the size guess was short
            else:
                out.append((offs[k].astype(np.int64), bufs[k][: int(totals[k])]))
        if info is not None:
            info["h2d_bytes"] = int(h2d.value)
            info["totals"] = [int(t) for t in totals]
            si = (ctypes.c_uint64 * 4)()
            with self._lock:
                check(lib.mdrq_stream_info(self.handle, si))
            # device->host bytes of the call and how many of its batches left
            # the device packed (16-bit low halves + bucket ends, pack.cu)
            info["d2h_bytes"] = int(si[0])
            info["packed_batches"] = int(si[1])
            info["packed_share"] = int(si[3]) / 1000.0   # of a packed batch's queries; the rest travel raw
        return out

    def stats(self, nq: int, mode: int = _lib.MODE_SCALAR):
        arr = (_lib.SearchStatsC * max(nq, 1))()
        with self._lock:
            check(_lib.load().mdrq_query_stats(self.handle, mode, arr, nq))
        return [arr[i] for i in range(nq)]

    # -- prepared batches (device-resident; bench / multi-GPU) --------------
    def prepare(self, lower, upper, path: str | int = "auto") -> "PreparedBatch":
        b = PreparedBatch(self, lower, upper, path)
        self._batches.add(b)
        return b


def _guess(n: int, nq: int) -> int:
    return int(min(max(4096, n // 64 * max(nq, 1)), 1 << 26))


def _path(path) -> int:
    if isinstance(path, str):
        try:
            return _lib.PATHS[path]
        except KeyError:
            raise ValueError(f"unknown path {path!r} (choose from {sorted(_lib.PATHS)})") from None
    return int(path)


class PreparedBatch:
    """A query batch whose descriptors live in HBM (``mdrq_batch``)."""

    def __init__(self, store: DeviceStore, lower, upper, path="auto"):
        lib = _lib.load()
        lo, hi = _bounds(lower, upper, store.m)
        self.store = store
        self.nq = lo.shape[0]
        h = ctypes.c_void_p()
        check(lib.mdrq_batch_prepare(store.handle, lo.ctypes.data_as(f32p), hi.ctypes.data_as(f32p),
                                     self.nq, _path(path), ctypes.byref(h)))
        self._h = h

    def close(self):
        h, self._h = getattr(self, "_h", None), None
        if h:
            # safe after the store is gone too: the store detached it
            _lib.load().mdrq_batch_destroy(h)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def count_async(self, d_counts: int = 0, stream: int = 0) -> None:
        check(_lib.load().mdrq_batch_count_async(self.store.handle, self._h, ctypes.c_void_p(d_counts or None),
                                                 ctypes.c_void_p(stream or None)))

    def ids_async(self, stream: int = 0) -> None:
        check(_lib.load().mdrq_batch_ids_async(self.store.handle, self._h, ctypes.c_void_p(stream or None)))

    def reserve(self) -> int:
        t = ctypes.c_uint64(0)
        check(_lib.load().mdrq_batch_reserve(self.store.handle, self._h, ctypes.byref(t)))
        return int(t.value)

    def result_device(self):
        """(device ptr of ids u32, device ptr of offsets u64[nq+1], total)."""
        a, b, t = ctypes.c_uint64(0), ctypes.c_uint64(0), ctypes.c_uint64(0)
        check(_lib.load().mdrq_result_device(self.store.handle, ctypes.byref(a), ctypes.byref(b),
                                             ctypes.byref(t)))
        return int(a.value), int(b.value), int(t.value)

    CLASSES = ("scan", "compaction", "id_write", "setup")
    PATH_NAMES = {v: k for k, v in _lib.PATHS.items()}

    def info(self) -> dict:
        arr = (ctypes.c_uint32 * 4)()
        check(_lib.load().mdrq_batch_info(self._h, arr))
        return {"path": self.PATH_NAMES.get(int(arr[0]), str(arr[0])), "nq": int(arr[1]),
                "passes": int(arr[2]), "max_union_dims": int(arr[3])}

    def profile(self, ids: bool, stream: int = 0) -> dict:
        """One synchronising pass with CUDA events between launch groups:
        {class: (device ms, kernel launches)}."""
        ms = (ctypes.c_double * 4)()
        nl = (ctypes.c_uint32 * 4)()
        check(_lib.load().mdrq_batch_profile(self.store.handle, self._h, int(bool(ids)),
                                             ctypes.c_void_p(stream or None), ms, nl))
        return {c: (float(ms[i]), int(nl[i])) for i, c in enumerate(self.CLASSES)}

    def launches(self, ids: bool) -> int:
        c = ctypes.c_uint32(0)
        check(_lib.load().mdrq_batch_launches(self._h, int(bool(ids)), ctypes.byref(c)))
        return int(c.value)
