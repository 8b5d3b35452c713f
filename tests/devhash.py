"""Device-side checker of a large ids result (TEST INFRASTRUCTURE).

A full-size configuration produces up to ~5e9 ids per batch (C5 ids mode:
20 GB); comparing it with the oracle on the host would move it over PCIe
and through numpy.  Instead the result is checked where it lies, with plain
torch arithmetic (not the product's kernels):

* every query's ids are strictly ascending and < n (so the list is fixed by
  its set), and
* per query (count, set hash) with hash = sum of splitmix64(id) mod 2**64 --
  exactly what the CPU oracle records in tests/golden/all_<cfg>.npz
  (oracle/mdrq_oracle.c ``oracle_hash_batch``).
"""

from __future__ import annotations

import numpy as np

_C = [0x9E3779B97F4A7C15, 0xBF58476D1CE4E5B9, 0x94D049BB133111EB]
_C = [c - (1 << 64) if c >= 1 << 63 else c for c in _C]   # as int64 (two's complement)


def _lsr(z, s):
    """Logical right shift of int64 (torch's >> is arithmetic)."""
    return (z >> s) & ((1 << (64 - s)) - 1)


def mix64(x):
    """splitmix64 finalizer on an int64 tensor, wrapping like uint64."""
    z = x + _C[0]
    z = (z ^ _lsr(z, 30)) * _C[1]
    z = (z ^ _lsr(z, 27)) * _C[2]
    return z ^ _lsr(z, 31)


def wrap(ptr: int, count: int, dtype, device):
    """A torch view of device memory (no copy)."""
    import torch
    typestr = {torch.int32: "<i4", torch.int64: "<i8"}[dtype]

    class _CAI:
        __cuda_array_interface__ = {"shape": (int(count),), "typestr": typestr, "data": (int(ptr), False),
                                    "version": 3, "strides": None}
    return torch.as_tensor(_CAI(), device=device)


def check_result(ids, offs, n_limit: int, chunk: int = 1 << 27):
    """(counts int64[nq], hashes uint64[nq]) of a result held in torch
    tensors (ids int32 holding uint32 ids, offs int64[nq+1]; any device),
    after asserting ascending ids < n_limit within every query."""
    import torch
    nq = offs.numel() - 1
    total = int(offs[-1])
    assert int(offs[0]) == 0
    counts = offs[1:] - offs[:-1]
    assert bool((counts >= 0).all())
    P = torch.zeros(nq + 1, dtype=torch.int64, device=offs.device)   # hash prefix at every offset
    carry = torch.zeros((), dtype=torch.int64, device=offs.device)
    for a in range(0, total, chunk):
        b = min(total, a + chunk)
        x = ids[a:b].to(torch.int64) & 0xFFFFFFFF
        assert int(x.max()) < n_limit, "id out of range"
        # ascending inside queries: a non-increasing step must sit at a query start
        lo_ = max(a - 1, 0)
        xx = ids[lo_:b].to(torch.int64) & 0xFFFFFFFF
        bad = torch.nonzero(xx[1:] <= xx[:-1]).flatten() + lo_ + 1   # i with id[i] <= id[i-1]
        if bad.numel():
            assert bool(torch.isin(bad, offs).all()), "ids not strictly ascending within a query"
        cs = torch.cumsum(mix64(x), 0) + carry
        sel = (offs > a) & (offs <= b)
        P[sel] = cs[offs[sel] - a - 1]
        carry = cs[-1]
    h = (P[1:] - P[:-1]).cpu().numpy().view(np.uint64)
    return counts.cpu().numpy(), h


def check_device_result(d_ids: int, d_offsets: int, nq: int, total: int, n_limit: int, device: int = 0):
    """check_result on a device result (uint32 ids at d_ids, uint64
    offsets[nq+1] at d_offsets) in place."""
    import torch
    dev = torch.device("cuda", device)
    offs = wrap(d_offsets, nq + 1, torch.int64, dev).clone()
    assert int(offs[-1]) == total
    ids = wrap(d_ids, max(total, 1), torch.int32, dev)
    return check_result(ids, offs, n_limit)


def batch_hashes(store, lo, hi, path: str, device: int = 0):
    """Run (lo, hi) as one prepared ids batch on `path` and check it on the
    device: -> (counts, hashes, path the planner ran)."""
    b = store.prepare(lo, hi, path)
    try:
        total = b.reserve()
        d_ids, d_offs, tot = b.result_device()
        assert tot == total
        counts, hashes = check_device_result(d_ids, d_offs, lo.shape[0], total, store.id_base + store.n, device)
        return counts, hashes, b.info()["path"]
    finally:
        b.close()
