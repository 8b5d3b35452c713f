"""B200-native MDRQ scan engine -- drop-in for the scan / VA-file hot path
of the reference ``mdrq`` package (arXiv 1801.03644).

The public names mirror /root/reference/pkg/src/mdrq/__init__.py for the
hot path: build from an (n, m) float32 array, query per-dimension
inclusive ``[lo, hi]`` boxes (with +-inf sentinels for unqueried
dimensions), get ascending ids or a count.  All compute runs in
``libmdrq_b200.so`` (hand-written sm_100a CUDA behind a C ABI,
include/mdrq_b200.h); there is no CPU fallback.  Tree indexes (kd-tree,
R*-tree) are out of scope.
"""

from . import _lib
from .core import (
    DataSet,
    KernelMode,
    RangeQuery,
    ResultSet,
    SearchStats,
    SelectivityStats,
    match,
    match_scalar,
    match_vectorized,
    read_dataset,
    selectivity_oracle,
    stack_queries,
    write_dataset,
)
from .kernels import BACKEND
from .methods import METHOD_NAMES, build_method
from .parallel import (
    PartitionLayout,
    ShardedScan,
    combine_counts,
    combine_ids,
    default_threads,
    make_layout,
    shard_range,
)
from .scan import (
    BatchResult,
    ColumnSet,
    HorizontalScan,
    SequentialScan,
    VerticalScan,
    horizontal_scan,
    sequential_scan,
    vertical_scan,
)
from .store import DeviceStore, PreparedBatch
from .vafile import QuantileGrid, VaFile
from .workload import (
    GeneratorSpec,
    gen_dataset,
    gen_query_from_pair,
    gen_uniform,
    pair_query_batch,
    read_queries,
    write_queries,
)

__version__ = "0.1.0"


def device_count() -> int:
    """CUDA devices visible to the engine (0 on a CPU-only host)."""
    return _lib.device_count()
