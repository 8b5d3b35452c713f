"""Row partitioning and multi-GPU fan-out / fan-in.

Reference: /root/reference/pkg/src/mdrq/parallel.py -- a seeded random
layout of p near-equal row partitions (make_layout, parallel.py:98-118),
one worker task per partition (WorkerPool, parallel.py:45-78) and a
concatenate + sort merge (PartitionedIndex, parallel.py:126-167).

On B200 the partitions are GPUs, one process per GPU:

* rows are split into CONTIGUOUS shards ``[r*ceil(n/W), ...)`` (``shard_range``)
  so a shard's local id + its start is the global id and rank-order
  concatenation is already sorted (no sort);
* each rank scans its shard with the device kernels;
* counts are combined with one all_gather; ids with an all_gather of the
  per-query counts followed by an all_gather of the (padded) id buffers and a
  vectorised scatter into rank order.  Over NCCL this runs on NVLink; the
  same functions run over gloo on CPU tensors for the tests.

``make_layout`` / ``PartitionLayout`` keep the reference's host-side API
(HorizontalScan and build_method accept layouts); the reference's thread
pool has no counterpart -- on one GPU the CTA grid is the fan-out.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np


def default_threads() -> int:
    """Host worker count: MDRQ_THREADS when it is a positive integer, else the
    logical core count (parallel.py:20-27).  On this engine it only sizes
    host-side helpers; the scan's parallelism is the CTA grid."""
    try:
        t = int(os.environ.get("MDRQ_THREADS", ""))
    except ValueError:
        t = 0
    return t if t >= 1 else (os.cpu_count() or 1)


@dataclass(frozen=True)
class PartitionLayout:
    """The reference's seeded row partitioning (parallel.py:81-118), kept so
    layout-taking constructors (HorizontalScan) accept the same arguments.
    ``parts[q]`` are the ids of partition q in permutation order and
    ``assignment[i]`` is the partition of object i.  The GPU scan does not
    need it (one store covers all rows); results do not depend on it."""

    p: int
    seed: int
    assignment: np.ndarray
    parts: tuple

    @property
    def n(self) -> int:
        return len(self.assignment)

    def sizes(self) -> list[int]:
        return [len(ids) for ids in self.parts]


def make_layout(n: int, p: int, seed: int) -> PartitionLayout:
    """``default_rng(seed).permutation(n)`` cut into p runs whose sizes differ
    by at most one, the larger runs first (parallel.py:98-118)."""
    if p < 1:
        raise ValueError("partition count must be at least 1")
    order = np.random.default_rng(seed).permutation(n).astype(np.int64)
    sizes = np.full(p, n // p, dtype=np.int64)
    sizes[: n % p] += 1
    cuts = np.cumsum(sizes)[:-1]
    assignment = np.empty(n, dtype=np.int32)
    assignment[order] = np.repeat(np.arange(p, dtype=np.int32), sizes)
    return PartitionLayout(p=p, seed=seed, assignment=assignment, parts=tuple(np.split(order, cuts)))


# ----------------------------------------------------------- GPU sharding --

def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous row shard [start, stop) of `rank` among `world` GPUs."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    per = -(-n // world)
    start = min(rank * per, n)
    return start, min(start + per, n)


def combine_counts(local_counts, group=None):
    """Sum per-query counts over ranks (one all_gather).  Tensor in, tensor out."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    local_counts = local_counts.to(torch.int64).contiguous().reshape(-1)
    return _all_gather(local_counts, world, group).sum(0)


def _all_gather(t, world: int, group):
    """[numel] -> [world, numel] (flat output: works on NCCL and gloo)."""
    import torch
    import torch.distributed as dist
    out = torch.empty(world * t.numel(), dtype=t.dtype, device=t.device)
    dist.all_gather_into_tensor(out, t, group=group)
    return out.view(world, t.numel())


def global_layout(all_counts):
    """all_counts [world, nq] (ids of query q on rank r) -> (out_offsets
    int64[nq+1] of the merged result, rank_prefix [world, nq]: where rank r's
    slice of query q starts inside query q's run).  Rank order is id order
    (contiguous shards), so the merge is the reference's concat + sort
    (scan.py:160, parallel.py:156-157) without the sort."""
    import torch
    nq = all_counts.shape[1]
    out_offsets = torch.zeros(nq + 1, dtype=torch.int64, device=all_counts.device)
    torch.cumsum(all_counts.sum(0), 0, out=out_offsets[1:])
    rank_prefix = torch.cumsum(all_counts, 0) - all_counts
    return out_offsets, rank_prefix


def rank_segments(all_counts, rank: int, out_offsets, rank_prefix):
    """Segments (src_off, dst_off, len), one per query, that place rank
    `rank`'s local result (query-major) into the merged query-major result."""
    import torch
    c = all_counts[rank]
    src_off = torch.cumsum(c, 0) - c
    dst_off = out_offsets[:-1] + rank_prefix[rank]
    return src_off.contiguous(), dst_off.contiguous(), c.contiguous()


def _place_segments(src, dst, src_off, dst_off, seg_len, stream=None):
    """dst[dst_off[i] : +len[i]] = src[src_off[i] : +len[i]] for every
    segment: one mdrq_copy_segments kernel when src lives on a GPU (dst may be
    device memory or registered host memory the device can write), torch
    index arithmetic on CPU tensors (the gloo tests)."""
    import torch
    nseg = seg_len.numel()
    if nseg == 0 or int(seg_len.sum()) == 0:
        return
    if src.device.type == "cuda" and src.element_size() == 4:
        import ctypes
        from . import _lib
        dptr = dst.data_ptr() if hasattr(dst, "data_ptr") else int(dst)
        st = stream if stream is not None else torch.cuda.current_stream(src.device).cuda_stream
        _lib.check(_lib.load().mdrq_copy_segments(
            ctypes.c_void_p(src.data_ptr()), ctypes.c_void_p(dptr),
            ctypes.c_void_p(src_off.data_ptr()), ctypes.c_void_p(dst_off.data_ptr()),
            ctypes.c_void_p(seg_len.data_ptr()), nseg, ctypes.c_void_p(st)))
        return
    total = int(seg_len.sum())
    base_dst = torch.repeat_interleave(dst_off - src_off, seg_len)
    src_idx = torch.repeat_interleave(src_off, seg_len)
    within = torch.arange(total, dtype=torch.int64, device=src.device) - torch.repeat_interleave(
        torch.cumsum(seg_len, 0) - seg_len, seg_len)
    dst[base_dst + src_idx + within] = src[src_idx + within]


def combine_ids(local_offsets, local_ids, group=None):
    """Rank-ordered merge of per-rank id lists.

    ``local_offsets`` int64[nq+1] and ``local_ids`` (global ids of this rank's
    shard, ascending per query) -> (offsets int64[nq+1], ids) identical on
    every rank (NCCL all_gather of the padded slices + one placement kernel).
    """
    import torch
    world = dist_world(group)
    dev = local_ids.device
    local_offsets = local_offsets.to(device=dev, dtype=torch.int64)
    counts = local_offsets[1:] - local_offsets[:-1]
    all_counts = _all_gather(counts.contiguous(), world, group)
    out_offsets, rank_prefix = global_layout(all_counts)
    maxlen = int(all_counts.sum(1).max().item()) if world else 0
    padded = torch.zeros(max(maxlen, 1), dtype=local_ids.dtype, device=dev)
    if local_ids.numel():
        padded[:local_ids.numel()] = local_ids
    gathered = _all_gather(padded, world, group)
    out = torch.empty(int(out_offsets[-1].item()), dtype=local_ids.dtype, device=dev)
    stride = gathered.shape[1]
    for r in range(world):
        src_off, dst_off, seg = rank_segments(all_counts, r, out_offsets, rank_prefix)
        _place_segments(gathered.reshape(-1)[r * stride:(r + 1) * stride], out, src_off, dst_off, seg)
    return out_offsets, out


def dist_world(group=None) -> int:
    import torch.distributed as dist
    return dist.get_world_size(group)


class SharedHostBuffer:
    """One host buffer mapped by every rank of the node (POSIX shared
    memory), registered with CUDA in every rank that has a device, so each
    rank's kernel writes its slices straight into it over its own PCIe link
    (rank-ordered offsets; no NCCL exchange of the ids, no second copy)."""

    def __init__(self, nbytes: int, group=None, device: int | None = None):
        import torch.distributed as dist
        from multiprocessing import shared_memory
        self.nbytes = max(int(nbytes), 1)
        rank = dist.get_rank(group)
        name = [None]
        if rank == 0:
            self._shm = shared_memory.SharedMemory(create=True, size=self.nbytes)
            name = [self._shm.name]
        dist.broadcast_object_list(name, src=dist.get_global_rank(group, 0) if group is not None else 0,
                                   group=group)
        if rank != 0:
            self._shm = shared_memory.SharedMemory(name=name[0])
        self.group = group
        self.rank = rank
        self._registered = False
        import numpy as _np
        self._arr = _np.ndarray((self.nbytes,), _np.uint8, buffer=self._shm.buf)
        if device is not None:
            import torch
            rc = torch.cuda.cudart().cudaHostRegister(self._arr.ctypes.data, self.nbytes, 3)  # portable | mapped
            if int(rc) != 0:
                raise RuntimeError(f"cudaHostRegister failed ({rc})")
            self._registered = True
        dist.barrier(group)

    @property
    def ptr(self) -> int:
        return int(self._arr.ctypes.data)

    def view(self, dtype, count: int):
        import numpy as _np
        return _np.ndarray((int(count),), dtype, buffer=self._shm.buf)

    def close(self):
        import torch.distributed as dist
        if getattr(self, "_shm", None) is None:
            return
        if self._registered:
            import torch
            torch.cuda.cudart().cudaHostUnregister(self._arr.ctypes.data)
            self._registered = False
        self._arr = None
        dist.barrier(self.group)
        self._shm.close()
        if self.rank == 0:
            self._shm.unlink()
        self._shm = None


def _dma_segments(local_ids, buf_ptr: int, src_off, dst_off, seg) -> bool:
    """Every segment device -> host with the copy engines (one async copy per
    segment, mdrq_copy_segments_dma) on a side stream ordered after the
    current one; False when the runtime refuses it."""
    import ctypes
    import torch
    from . import _lib
    so = src_off.cpu().numpy().astype(np.int64)
    do = dst_off.cpu().numpy().astype(np.int64)
    sl = seg.cpu().numpy().astype(np.int64)
    dev = local_ids.device
    side = torch.cuda.Stream(dev)
    side.wait_stream(torch.cuda.current_stream(dev))
    p64 = ctypes.POINTER(ctypes.c_int64)
    rc = _lib.load().mdrq_copy_segments_dma(ctypes.c_void_p(local_ids.data_ptr()), ctypes.c_void_p(buf_ptr),
                                            so.ctypes.data_as(p64), do.ctypes.data_as(p64), sl.ctypes.data_as(p64),
                                            so.size, ctypes.c_void_p(side.cuda_stream))
    side.synchronize()
    return rc == 0


def gather_ids_to_host(local_offsets, local_ids, group=None, out: SharedHostBuffer | None = None,
                       method: str = "dma"):
    """Merged ids of every rank in ONE host buffer, written by the ranks
    themselves: the per-query counts are all_gathered (8 B per query and
    rank), every rank computes where its slice of each query goes and copies
    it there (on a GPU: one placement kernel into the registered shared host
    buffer, i.e. each rank's own PCIe link; on CPU: torch indexing).
    -> (offsets int64[nq+1] numpy, ids uint32 numpy view of the shared
    buffer, the buffer).  Rank order = id order, so no sort."""
    import numpy as _np
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = local_ids.device
    local_offsets = local_offsets.to(device=dev, dtype=torch.int64)
    counts = local_offsets[1:] - local_offsets[:-1]
    all_counts = _all_gather(counts.contiguous(), world, group)
    out_offsets, rank_prefix = global_layout(all_counts)
    total = int(out_offsets[-1].item())
    buf = out if out is not None else SharedHostBuffer(4 * total, group,
                                                       device=dev.index if dev.type == "cuda" else None)
    if buf.nbytes < 4 * total:
        raise ValueError(f"host buffer holds {buf.nbytes // 4} ids, the merge needs {total}")
    src_off, dst_off, seg = rank_segments(all_counts, rank, out_offsets, rank_prefix)
    if dev.type == "cuda":
        # the copy engines (DMA, ~the pinned-copy bandwidth of the link), else
        # the placement kernel writing through the mapping
        if method != "dma" or not _dma_segments(local_ids, buf.ptr, src_off, dst_off, seg):
            _place_segments(local_ids, buf.ptr, src_off, dst_off, seg)
            torch.cuda.current_stream(dev).synchronize()
    else:
        host = torch.from_numpy(buf.view(_np.int32, total)) if total else torch.empty(0, dtype=torch.int32)
        _place_segments(local_ids.to(torch.int32), host, src_off, dst_off, seg)
    dist.barrier(group)
    return out_offsets.cpu().numpy(), buf.view(_np.uint32, total), buf


class ShardedScan:
    """One rank's part of a row-sharded scan over W GPUs (one process each),
    the analog of the reference's PartitionedIndex (parallel.py:126-167):
    fan-out = every rank scans its contiguous shard, fan-in = the rank-ordered
    merge (no sort).  Results of ``count_batch`` / ``search_batch`` are
    global and identical on every rank; ``search_batch_host`` leaves the
    merged ids in one node-shared host buffer written by every rank directly.

    ``store`` may be any object with the DeviceStore query interface (the
    gloo tests inject the CPU oracle scan of the shard); by default a
    DeviceStore over ``shard_values`` with ``id_base`` = the shard start.
    """

    def __init__(self, shard_values, start: int, n_total: int, *, group=None, path: str = "auto",
                 layouts=None, va_bits: int = 8, device: int | None = None, store=None):
        from . import _lib
        from .store import DeviceStore
        self.group = group
        self.start = int(start)
        self.n_total = int(n_total)
        self.path = path
        if store is None:
            if layouts is None:
                layouts = _lib.LAYOUT_COLUMNAR | _lib.LAYOUT_VAFILE
            store = DeviceStore(shard_values, layouts=layouts, va_bits=va_bits, device=device, id_base=self.start)
        self.store = store
        self.m = store.m

    def _comm_device(self):
        import torch
        import torch.distributed as dist
        if dist.get_backend(self.group) == "nccl":
            return torch.device("cuda", self.store.device)
        return torch.device("cpu")

    def count_batch(self, lower, upper, path: str | None = None):
        import torch
        local = self.store.count(lower, upper, path or self.path)
        return combine_counts(torch.as_tensor(local, device=self._comm_device()), self.group).cpu().numpy()

    def _local(self, lower, upper, path):
        """This shard's result as tensors on the communication device; on a
        GPU the ids stay in HBM (a prepared batch, its pool read in place)."""
        import torch
        dev = self._comm_device()
        if dev.type == "cuda" and hasattr(self.store, "prepare"):
            b = self.store.prepare(lower, upper, path or self.path)
            try:
                total = b.reserve()
                d_ids, d_offs, _ = b.result_device()
                ids = _wrap_device(d_ids, total, torch.int32, dev).clone()
                offs = _wrap_device(d_offs, b.nq + 1, torch.int64, dev).clone()
            finally:
                b.close()
            return offs, ids
        offs, ids = self.store.ids(lower, upper, path or self.path)
        return (torch.as_tensor(np.asarray(offs, np.int64), device=dev),
                torch.as_tensor(np.asarray(ids).astype(np.int32, copy=False), device=dev))

    def search_batch(self, lower, upper, path: str | None = None):
        """-> (offsets int64[nq+1], ids uint32), the whole table's result."""
        offs, ids = self._local(lower, upper, path)
        o, i = combine_ids(offs, ids, self.group)
        return o.cpu().numpy(), i.cpu().numpy().view(np.uint32)

    def search_batch_host(self, lower, upper, path: str | None = None, out: SharedHostBuffer | None = None):
        """-> (offsets, ids uint32 view of the shared host buffer, buffer):
        every rank writes its own slices (SharedHostBuffer); the caller
        closes the buffer when done with the ids."""
        offs, ids = self._local(lower, upper, path)
        return gather_ids_to_host(offs, ids, self.group, out)

    def close(self):
        self.store.close()


def _wrap_device(ptr: int, count: int, dtype, dev):
    """Device pointer -> torch tensor (no copy)."""
    import torch
    typestr = {torch.int32: "<i4", torch.int64: "<i8"}[dtype]

    class _CAI:
        __cuda_array_interface__ = {"shape": (int(count),), "typestr": typestr, "data": (int(ptr), False),
                                    "version": 3, "strides": None}
    return torch.as_tensor(_CAI(), device=dev)
