"""B200-native (sm_100a) PaLD cohesion engine.

Drop-in GPU implementation of the O(n^3) hot path of the PaLD reference
library (arXiv 2307.16652): local-focus sizes u_xy and cohesion updates for
the pairwise and triplet algorithms. The C ABI (include/pald_gpu.h) is the
boundary; this package mirrors the reference API on top of it.
"""
from .api import (  # noqa: F401
    CohesionMatrix,
    DistanceMatrix,
    Error,
    FocusSizeMatrix,
    GpuError,
    IoError,
    LocalDepthVector,
    PaldResult,
    ParallelPlan,
    PhaseTimes,
    Policy,
    UnsupportedPolicyError,
    UpdateStyle,
    ValidationError,
    blocked_pairwise,
    blocked_triplet,
    fill_diagonal,
    local_depths,
    normalize,
    parallel_pairwise,
    parallel_triplet,
    to_string,
)

__version__ = "0.1.0"


def build(force: bool = False):
    from ._build import build as _b

    return _b(force=force)
