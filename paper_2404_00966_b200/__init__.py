"""B200-native GTS batch similarity search (arXiv 2404.00966).

Drop-in for the reference package's hot path (`metrictree`: build,
BatchSearcher.range_batch / knn_batch, StreamingIndex): the same Python
surface, backed by hand-written sm_100a CUDA kernels in libgts.so behind a
C ABI (include/gts.h).
"""

from .data import DataObject, Dataset, generate_clustered, generate_sequences, generate_uniform
from .metrics import (
    ANGULAR,
    EDIT,
    L1,
    L2,
    METRIC_KINDS,
    MetricMismatchError,
    distance,
    edit_distance,
    pair_distances,
)
from .runtime import DEFAULT_MEMORY_UNITS, BudgetError, MemoryBudget, ParallelRuntime
from .search import (
    BatchSearcher,
    CsrResult,
    SearchStats,
    compute_query_groups,
    current_kth_bound,
    level_size_limit,
    node_prunable_knn,
    node_prunable_range,
    object_prunable,
)
from .tree import (
    ConfigError,
    FlatPivotTree,
    TreeConfig,
    build,
    child_node_id,
    decode_distance,
    encode_distance,
    level_range,
    parent_node_id,
    tree_height,
)
from .snapshot import SnapshotFormatError, load_snapshot, save_snapshot
from .updates import StreamingIndex, UpdateError

__version__ = "0.1.0"

__all__ = [
    "SnapshotFormatError", "load_snapshot", "save_snapshot",
    "ANGULAR", "EDIT", "L1", "L2", "METRIC_KINDS", "BatchSearcher", "BudgetError", "ConfigError",
    "CsrResult", "DataObject", "Dataset", "DEFAULT_MEMORY_UNITS", "FlatPivotTree", "MemoryBudget",
    "MetricMismatchError", "ParallelRuntime", "SearchStats", "StreamingIndex", "TreeConfig", "UpdateError",
    "build", "child_node_id", "compute_query_groups", "current_kth_bound", "decode_distance", "distance",
    "edit_distance", "encode_distance", "generate_clustered", "generate_sequences", "generate_uniform",
    "level_range", "level_size_limit", "node_prunable_knn", "node_prunable_range", "object_prunable",
    "pair_distances", "parent_node_id", "tree_height",
]
