"""B200-native sliding super point detector (arXiv 1803.11036).

The product is the CUDA library lib/libsspd_cuda.so behind the C ABI in
include/sspd_cuda.h, plus the C++ drop-in of the reference's sspd:: API
(lib/libsspd.so, headers in include/sspd/).  This package is the Python view
of the same C ABI used by the tests, the bench and torch.distributed
multi-router runs.
"""
from ._cabi import (CandidateOverflow, CudaError, InvalidArgument, NoDevice, OutOfRange,
                    PAPER_MAX, UNION_MIN, SspdError, load)
from .grid import (BASE_NOW, Detection, Grid, checked_status, device_count, device_ordinals, estimate_cardinality, exact_counts,
                   export_snapshot,
                   hot_cutoff, import_snapshot, launch_count, merge_rseas, release_cached)

from .pipeline import run_detection, validate_config
from .trace import read_trace, write_trace

__all__ = [
    "run_detection", "validate_config", "read_trace", "write_trace",
    "BASE_NOW", "CandidateOverflow", "CudaError", "Detection", "Grid", "InvalidArgument",
    "NoDevice", "OutOfRange", "PAPER_MAX", "SspdError", "UNION_MIN", "checked_status", "device_count", "device_ordinals",
    "estimate_cardinality", "exact_counts", "export_snapshot", "hot_cutoff", "import_snapshot", "launch_count",
    "load", "merge_rseas", "release_cached",
]
