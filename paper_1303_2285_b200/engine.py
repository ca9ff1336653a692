"""Front end: the reference's covariance entry points, executed on the GPU.

Signatures, argument validation and exception types follow the reference
engine (``engine.py:108-255``); the body of every entry point is one call
into libcovgpu.so (``include/covgpu.h``) instead of the per-class thread pool
(``engine.py:158-190``).  The CPU execution modes of the reference ("seq",
"seq-opt", "par" with ``threads``) are accepted and validated, and all run
the same GPU path; as in the reference (``test_engine.py:79-108``) the result
is bitwise independent of mode, thread count and dispatch order.

Unlike the reference, results are normalised by 1/K and returned as a dense
Hermitian device tensor (BASELINE.json north_star).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _native
from . import combinations as _comb
from .core import CovarianceMatrix, InputMatrix, WindowSpec, _to_device_matrix, packed_size

__all__ = [
    "MODE_SEQ_DIRECT",
    "MODE_SEQ_OPTIMIZED",
    "MODE_PARALLEL",
    "BACKEND",
    "OpCounters",
    "resolve_backend",
    "estimate_combinations",
    "estimate_seq_direct",
    "estimate_seq_optimized",
    "estimate_parallel",
    "estimate_batch",
    "estimate_batch_tensor",
    "estimate_tensor",
]

MODE_SEQ_DIRECT = "seq"
MODE_SEQ_OPTIMIZED = "seq-opt"
MODE_PARALLEL = "par"
BACKEND = "cuda"

_DTYPE_CODE = {torch.complex128: _native.C128, torch.complex64: _native.C64}


@dataclass(frozen=True)
class OpCounters:
    """Exact operation counts of one estimate (``engine.py:42-75``).

    multiplications = sum of mu over UC = UM (Eq. 4.6) — every product is
    formed exactly once (the paper's count; the default spectral engine gets
    the same sums with far fewer hardware multiplies).  additions is a MODEL,
    not a count of executed instructions: one accumulate per product plus two
    per slot for the diagonal-segment walk — the direct CUDA-core kernels'
    arithmetic (the reference's figure is backend-specific too).
    """

    multiplications: int
    additions: int
    per_combination: tuple

    @classmethod
    def tally(cls, combos, window: WindowSpec, n: int, m: int) -> "OpCounters":
        per = []
        for comb in combos:
            mults = _comb.pair_count(comb, n, m)
            adds = mults + 2 * _comb.max_writes(comb, window)
            per.append((comb, mults, adds))
        return cls(
            multiplications=sum(r[1] for r in per),
            additions=sum(r[2] for r in per),
            per_combination=tuple(per),
        )


def resolve_backend(name: str | None = None) -> str:
    """The single execution path.  Replaces ``backend.resolve_backend``
    (``backend.py:45-57``): there is no multi-backend dispatch and no CPU
    fallback, so the CPU backends of the reference are refused."""
    choice = (name or "auto").strip().lower()
    if choice in ("auto", BACKEND):
        return BACKEND
    if choice in ("numba", "numpy"):
        raise RuntimeError(
            f"backend {name!r} is a CPU path of the reference; covgpu runs only on 'cuda'"
        )
    raise ValueError(f"unknown backend {name!r}; expected 'cuda' or 'auto'")


def _stream_ptr(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _run(stack: torch.Tensor, window: WindowSpec, class_ids=None, layout=_native.DENSE,
         out: torch.Tensor | None = None, scale: float | None = None) -> torch.Tensor:
    """One C-ABI call over a (B, N, M) device stack; returns R in `layout`."""
    b, n, m = stack.shape
    window.validate_for(n, m)
    dim = window.stack_size
    if packed_size(dim) > 2**31 - 1:
        raise ValueError(f"packed triangle of a {dim}x{dim} matrix exceeds 2^31-1 entries")
    lib = _native.lib()
    code = _DTYPE_CODE[stack.dtype]
    k = (n - window.p + 1) * (m - window.q + 1)
    ids, nids = _native.id_array(class_ids)
    elems = lib.covgpu_output_elems(b, n, m, window.p, window.q, layout, ids, nids)
    if elems < 0:
        raise ValueError("invalid output layout or class ids")
    if out is None:
        if layout == _native.DENSE:
            shape = (b, dim, dim)
        else:
            shape = (b, elems // b)
        alloc = torch.zeros if class_ids is not None else torch.empty
        out = alloc(shape, dtype=stack.dtype, device=stack.device)
    elif out.numel() != elems or out.dtype != stack.dtype or not out.is_contiguous():
        raise ValueError("out tensor has the wrong size, dtype or layout")
    with torch.cuda.device(stack.device):
        rc = lib.covgpu_estimate(
            ctypes.c_void_p(stack.data_ptr()), b, n, m, window.p, window.q, code, layout,
            ids, nids, 1.0 / k if scale is None else scale,
            ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(_stream_ptr(stack.device)),
        )
    _native.check(rc, "covgpu_estimate")
    return out


def estimate_tensor(a, window: WindowSpec, class_ids=None, device=None, dtype=None) -> torch.Tensor:
    """Dense normalised R (PQ x PQ device tensor) of one matrix — the fast path
    without result wrappers or counters."""
    t = _to_device_matrix(a, device, dtype, ndim=2)
    return _run(t.unsqueeze(0), window, class_ids)[0]


def estimate_combinations(
    a,
    window: WindowSpec,
    mode: str = MODE_SEQ_DIRECT,
    threads: int = 1,
    backend: str | None = None,
    sorted_dispatch: bool = True,
) -> tuple[CovarianceMatrix, OpCounters]:
    """Estimate the windowed covariance via the class decomposition
    (``engine.py:108-147``).  Returns the normalised estimate and the counters."""
    if mode == MODE_PARALLEL:
        return estimate_parallel(a, window, threads, backend=backend, sorted_dispatch=sorted_dispatch)
    if mode not in (MODE_SEQ_DIRECT, MODE_SEQ_OPTIMIZED):
        raise ValueError(f"unknown mode {mode!r}")
    resolve_backend(backend)
    mat = a if isinstance(a, InputMatrix) else InputMatrix(a)
    window.validate_for(mat.n, mat.m)
    dense = _run(mat.tensor.unsqueeze(0), window)[0]
    k = (mat.n - window.p + 1) * (mat.m - window.q + 1)
    counters = OpCounters.tally(_comb.unique_combinations(window), window, mat.n, mat.m)
    return CovarianceMatrix(dense, k), counters


def estimate_seq_direct(a, window: WindowSpec, backend: str | None = None):
    return estimate_combinations(a, window, MODE_SEQ_DIRECT, backend=backend)


def estimate_seq_optimized(a, window: WindowSpec, backend: str | None = None):
    return estimate_combinations(a, window, MODE_SEQ_OPTIMIZED, backend=backend)


def estimate_parallel(
    a,
    window: WindowSpec,
    threads: int = 1,
    backend: str | None = None,
    sorted_dispatch: bool = True,
) -> tuple[CovarianceMatrix, OpCounters]:
    """Thread-parallel entry point of the reference (``engine.py:193-216``);
    the GPU spreads classes over SMs itself, so `threads` is validated only."""
    if threads < 1:
        raise ValueError(f"threads must be >= 1, got {threads}")
    return estimate_combinations(a, window, MODE_SEQ_OPTIMIZED, backend=backend)


def estimate_batch_tensor(stack, window: WindowSpec, device=None, dtype=None) -> torch.Tensor:
    """(B, PQ, PQ) dense normalised estimates of a (B, N, M) stack in one launch set."""
    t = _to_device_matrix(stack, device, dtype, ndim=3)
    return _run(t, window)


def estimate_batch(
    matrices,
    window: WindowSpec,
    threads: int = 1,
    backend: str | None = None,
    sorted_dispatch: bool = True,
) -> list[CovarianceMatrix]:
    """Several same-sized matrices in one launch set (``engine.py:219-255``).

    Accepts a list of matrices (as the reference) or a 3-D (B, N, M) array or
    tensor.  Outputs equal per-matrix estimates bit for bit."""
    if threads < 1:
        raise ValueError(f"threads must be >= 1, got {threads}")
    resolve_backend(backend)
    if isinstance(matrices, torch.Tensor) and matrices.dim() == 3:
        stack = _to_device_matrix(matrices, None, None, ndim=3)
    else:
        if hasattr(matrices, "ndim") and getattr(matrices, "ndim") == 3:
            mats = [matrices[i] for i in range(matrices.shape[0])]
        else:
            mats = list(matrices)
        if not mats:
            raise ValueError("batch must contain at least one matrix")
        tens = [InputMatrix(x).tensor if not isinstance(x, InputMatrix) else x.tensor for x in mats]
        n, m = tens[0].shape
        for t in tens[1:]:
            if t.shape != (n, m):
                raise ValueError(
                    f"batch matrices must share dimensions; got {n}x{m} and {t.shape[0]}x{t.shape[1]}"
                )
        dtype = torch.complex64 if all(t.dtype == torch.complex64 for t in tens) else torch.complex128
        stack = torch.stack([t.to(dtype) for t in tens])
    b, n, m = stack.shape
    window.validate_for(n, m)
    dense = _run(stack, window)
    k = (n - window.p + 1) * (m - window.q + 1)
    return [CovarianceMatrix(dense[i], k) for i in range(b)]


def measure_unit_times(a, window: WindowSpec, repeats: int = 3, device=None):
    """Best-of-repeats GPU time of every bulk work unit (the partitioner's
    unit: one walk over A's rows for `lags` x `warps` classes), each run as a
    class-subset plan (edge rows and finalize of those classes included).
    Returns [(class ids, seconds)] in unit order."""
    from .partition import work_units
    from .plan import Plan

    if repeats < 1:
        raise ValueError(f"repeats must be >= 1, got {repeats}")
    t = _to_device_matrix(a, device, None, ndim=2)
    n, m = t.shape
    window.validate_for(n, m)
    units = work_units(n, m, window, fp64=t.dtype == torch.complex128)
    out = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a3 = t.unsqueeze(0)
    for ids, _cost in units:
        plan = Plan(n, m, window, dtype=t.dtype, class_ids=ids, device=t.device)
        dst = plan.alloc_output("compact")
        plan.execute(a3, dst, "compact")  # warm
        best = float("inf")
        for _ in range(repeats):
            e0.record()
            plan.execute(a3, dst, "compact")
            e1.record()
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1) * 1e-3)
        plan.close()
        out.append((ids, best))
    return out


def measure_combination_times(a, window: WindowSpec, backend: str | None = None, repeats: int = 3,
                              classes=None):
    """Per-class GPU cost in UC order, the reference's trace contract
    (``engine.py:258-288``: best-of-repeats wall time of each class kernel):
    every class is run ALONE as a one-class plan — its sums, edge sums and
    diagonal-segment walk, nothing apportioned — and timed with CUDA events
    around the plan's launches.  `classes` restricts the measurement to some
    UC indices (the others get None).  Feeds ``write_cost_trace`` and the
    reference's scheduling simulator (``schedsim.ingest_measured_costs``)."""
    from .plan import Plan

    resolve_backend(backend)
    if repeats < 1:
        raise ValueError(f"repeats must be >= 1, got {repeats}")
    t = _to_device_matrix(a, None, None, ndim=2)
    n, m = t.shape
    window.validate_for(n, m)
    combos = _comb.unique_combinations(window)
    todo = range(len(combos)) if classes is None else sorted(set(int(i) for i in classes))
    cost = [None] * len(combos)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a3 = t.unsqueeze(0)
    for i in todo:
        plan = Plan(n, m, window, dtype=t.dtype, class_ids=[i], device=t.device)
        dst = plan.alloc_output("compact")
        plan.execute(a3, dst, "compact")  # warm (attributes, graph capture on the next call)
        plan.execute(a3, dst, "compact")
        best = float("inf")
        for _ in range(repeats):
            e0.record()
            plan.execute(a3, dst, "compact")
            e1.record()
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1) * 1e-3)
        plan.close()
        cost[i] = best
    return [(combos[i], cost[i]) for i in range(len(combos))]


TRACE_HEADER = ["task_id", "dr", "dc", "cost"]


def write_cost_trace(path, entries) -> None:
    """(Combination, cost) pairs as the reference's trace CSV
    (``schedsim.py:164-171``, header task_id,dr,dc,cost)."""
    import csv

    with open(path, "w", newline="", encoding="utf-8") as fh:
        w = csv.writer(fh)
        w.writerow(TRACE_HEADER)
        for task_id, (comb, c) in enumerate(entries):
            w.writerow([task_id, comb.dr, comb.dc, repr(float(c))])
