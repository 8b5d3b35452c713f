"""Uniform access-method registry (reference methods.py:17-47) on the GPU.

``build_method(name, data, ...)`` keeps the reference's names and keyword
arguments; the scan and VA-file methods are GPU executors.  ``gpu_*`` names
are explicit aliases.  The tree indexes are out of scope for this engine
 and raise.
"""

from __future__ import annotations

from dataclasses import dataclass

from .core import DataSet, KernelMode
from .parallel import default_threads
from .scan import HorizontalScan, SequentialScan, VerticalScan
from .store import DEFAULT_VA_BITS
from .vafile import VaFile

METHOD_NAMES = ("sequential", "horizontal", "vertical", "vafile",
                "gpu_rowwise", "gpu_columnar", "gpu_vafile")
OUT_OF_SCOPE = ("kdtree", "rstar")


@dataclass(frozen=True)
class _ContiguousLayout:
    """Stand-in layout for build_method('horizontal'): the GPU scan shards
    contiguously, so materialising the reference's n-element permutation
    (parallel.py:98-118) would only cost host memory."""

    n: int
    p: int

    def sizes(self) -> list[int]:
        base, extra = divmod(self.n, self.p)
        return [base + (1 if q < extra else 0) for q in range(self.p)]


def build_method(name: str, data: DataSet, *, threads: int | None = None, partitions: int | None = None,
                 mode: KernelMode = KernelMode.SCALAR, seed: int = 0, rstar_config=None,
                 device: int | None = None, va_bits: int = DEFAULT_VA_BITS):
    """Build one access method over a dataset (methods.py:20-47)."""
    t = threads if threads is not None else default_threads()
    p = partitions if partitions is not None else t
    if name in ("sequential", "gpu_rowwise"):
        return SequentialScan(data, mode, device=device)
    if name == "horizontal":
        return HorizontalScan(data, _ContiguousLayout(data.n, p), mode=mode, threads=t, device=device)
    if name in ("vertical", "gpu_columnar"):
        return VerticalScan(data, threads=t, mode=mode, device=device)
    if name in ("vafile", "gpu_vafile"):
        return VaFile.from_dataset(data, mode=mode, bits=va_bits, device=device)
    if name in OUT_OF_SCOPE:
        raise ValueError(f"access method {name!r} is a tree index and out of scope for the GPU scan "
                         f"engine (choose from {METHOD_NAMES})")
    raise ValueError(f"unknown access method {name!r} (choose from {METHOD_NAMES})")
