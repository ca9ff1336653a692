"""paper_1303_2285_b200 — B200-native windowed covariance estimation.

Drop-in GPU path for the reference package ``covcomb``'s covariance entry
points (arXiv 1303.2285): R = (1/K) sum_{windows} x x^H for an N x M complex
matrix and a P x Q sliding window, computed by hand-written sm_100a CUDA
kernels (``csrc/covgpu.cu``) behind the C ABI in ``include/covgpu.h``.
"""

from .combinations import (
    Combination,
    class_index,
    is_unique_combination,
    max_writes,
    pair_count,
    um_count,
    unique_combinations,
    work_groups,
)
from .core import (
    MAX_PACKED_ENTRIES,
    CovarianceMatrix,
    InputMatrix,
    WindowSpec,
    as_input_matrix,
    column_stack_index,
    max_rel_diff,
    packed_offset,
    packed_size,
    rel_frobenius_distance,
)
from .engine import (
    MODE_PARALLEL,
    MODE_SEQ_DIRECT,
    MODE_SEQ_OPTIMIZED,
    OpCounters,
    estimate_batch,
    estimate_batch_tensor,
    estimate_combinations,
    estimate_parallel,
    estimate_seq_direct,
    estimate_seq_optimized,
    estimate_tensor,
    resolve_backend,
)

__version__ = "0.1.0"
