"""Multi-GPU driver: one process per GPU over torch.distributed (NCCL).

The path shards with no data-path collective: offset
classes are independent and own disjoint slots of R (the reference's
disjointness theorem, ``combinations.py:1-13``, ``test_acceptance.py:64-86``),
and batch snapshots are independent (``engine.py:219-255``).  So:

* ``estimate_sharded`` — the single large estimate (cfg5 shape): rank 0's A is
  broadcast, every rank computes the classes of its shard
  (``partition.partition_classes``, product-balanced, bitwise identical to the
  unsharded result), and — only when asked — the compact shards are gathered
  to rank 0, which scatters them into the dense Hermitian R.
* ``estimate_batch_sharded`` — the batched config (cfg4): snapshots are split
  contiguously across ranks; each rank returns its own (b, PQ, PQ) slice, and
  rank 0 can gather the full batch.

* ``estimate_rowband`` — the single large estimate on the tensor-core path:
  the sums the kernels accumulate (CC, edge-column and edge-row sums) are
  sums over A's rows, so each rank computes one row band of every sum
  (``covgpu_plan_execute_sums``), the bands meet in ONE all-reduce of the
  [CC | CCol | RC'] buffer (16 MB at cfg5), and each rank finalizes a
  contiguous, slot-balanced range of classes from the reduced sums
  (``covgpu_plan_finalize_sums``); rank 0 gathers the compact ranges on
  request.  Unlike class sharding, every rank keeps the tensor-core kernels.

The per-shard compute and the root-side scatter are injectable (``ShardOps``,
``BandOps``) so the orchestration can be tested on CPU with the gloo backend;
the default ops are the CUDA library and there is no CPU fallback.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import torch
import torch.distributed as dist

from .core import WindowSpec
from .partition import partition_classes

__all__ = ["ShardOps", "cuda_ops", "estimate_sharded", "estimate_batch_sharded", "shard_bounds",
           "BandOps", "cuda_band_ops", "estimate_rowband", "class_ranges"]


@dataclass
class ShardOps:
    # (A (N,M) tensor, window, class_ids) -> compact slots of those classes (1-D tensor)
    compute_compact: Callable
    # (list of compact tensors, list of class-id lists, window, N, M, dtype, device) -> dense R
    scatter_dense: Callable
    # (A (B,N,M) tensor, window) -> (B, PQ, PQ) dense R
    compute_batch: Callable


def cuda_ops() -> ShardOps:
    from . import _native
    from .engine import _run

    def compute_compact(a, window, ids):
        return _run(a.unsqueeze(0), window, class_ids=ids, layout=_native.COMPACT)[0]

    def scatter_dense(compacts, id_lists, window, n, m, dtype, device):
        import ctypes

        lib = _native.lib()
        dim = window.stack_size
        k = (n - window.p + 1) * (m - window.q + 1)
        out = torch.empty((dim, dim), dtype=dtype, device=device)
        code = _native.C128 if dtype == torch.complex128 else _native.C64
        for comp, ids in zip(compacts, id_lists):
            if not ids:
                continue
            arr, nids = _native.id_array(ids)
            rc = lib.covgpu_scatter_compact(
                ctypes.c_void_p(comp.data_ptr()), 1, n, m, window.p, window.q, code, arr, nids,
                ctypes.c_void_p(out.data_ptr()),
                ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream))
            _native.check(rc, "covgpu_scatter_compact")
        del k
        return out

    def compute_batch(a, window):
        return _run(a, window)

    return ShardOps(compute_compact, scatter_dense, compute_batch)


def _r(t: torch.Tensor) -> torch.Tensor:
    """Real view for collectives (gloo has no complex dtypes)."""
    return torch.view_as_real(t) if t.is_complex() else t


def _world():
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def estimate_sharded(a: torch.Tensor | None, shape: tuple[int, int], window: WindowSpec,
                     dtype=torch.complex128, device=None, gather: bool = False,
                     ops: ShardOps | None = None):
    """Class-sharded estimate of one matrix across the process group.

    `a` is the (N, M) input on rank 0 (ignored elsewhere).  Returns
    (dense R on rank 0 if `gather` else None, this rank's compact shard,
    this rank's class ids)."""
    ops = ops or cuda_ops()
    rank, world = _world()
    n, m = shape
    window.validate_for(n, m)
    if device is None:
        device = a.device if (a is not None and rank == 0) else torch.device("cpu")
    buf = a if rank == 0 else torch.empty((n, m), dtype=dtype, device=device)
    if world > 1:
        dist.broadcast(_r(buf), src=0)
    shards = partition_classes(n, m, window, world)
    ids = shards[rank]
    comp = ops.compute_compact(buf, window, ids) if ids else torch.empty(0, dtype=dtype, device=device)
    dense = None
    if gather:
        if world > 1:
            sizes = [None] * world
            dist.all_gather_object(sizes, int(comp.numel()))
            width = max(sizes)
            padded = torch.zeros(width, dtype=dtype, device=device)
            padded[: comp.numel()] = comp
            bucket = [torch.empty_like(padded) for _ in range(world)] if rank == 0 else None
            dist.gather(_r(padded), [_r(x) for x in bucket] if rank == 0 else None, dst=0)
            if rank == 0:
                parts = [bucket[r][: sizes[r]] for r in range(world)]
                dense = ops.scatter_dense(parts, shards, window, n, m, dtype, device)
        else:
            dense = ops.scatter_dense([comp], [ids], window, n, m, dtype, device)
    return dense, comp, ids


def shard_bounds(batch: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous snapshot range of `rank` (sizes differ by at most one)."""
    base, extra = divmod(batch, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def estimate_batch_sharded(stack: torch.Tensor | None, shape: tuple[int, int, int],
                           window: WindowSpec, dtype=torch.complex64, device=None,
                           gather: bool = False, ops: ShardOps | None = None):
    """Snapshot-sharded batch estimate.  `stack` (B, N, M) lives on rank 0;
    each rank receives its slice (scatter), computes (b, PQ, PQ), and rank 0
    optionally gathers the full (B, PQ, PQ) batch.  Returns (full or None,
    local slice, (lo, hi))."""
    ops = ops or cuda_ops()
    rank, world = _world()
    batch, n, m = shape
    window.validate_for(n, m)
    if device is None:
        device = stack.device if (stack is not None and rank == 0) else torch.device("cpu")
    lo, hi = shard_bounds(batch, world, rank)
    local = torch.empty((hi - lo, n, m), dtype=dtype, device=device)
    if world > 1:
        # scatter by point-to-point (slices can differ in size by one)
        if rank == 0:
            reqs = []
            for r in range(1, world):
                rlo, rhi = shard_bounds(batch, world, r)
                if rhi > rlo:
                    reqs.append(dist.isend(_r(stack[rlo:rhi].contiguous()), dst=r))
            local.copy_(stack[lo:hi])
            for q in reqs:
                q.wait()
        elif hi > lo:
            dist.recv(_r(local), src=0)
    else:
        local.copy_(stack[lo:hi])
    out = ops.compute_batch(local, window) if hi > lo else torch.empty(
        (0, window.stack_size, window.stack_size), dtype=dtype, device=device)
    full = None
    if gather:
        dim = window.stack_size
        if world > 1:
            if rank == 0:
                full = torch.empty((batch, dim, dim), dtype=dtype, device=device)
                full[lo:hi] = out
                for r in range(1, world):
                    rlo, rhi = shard_bounds(batch, world, r)
                    if rhi > rlo:
                        dist.recv(_r(full[rlo:rhi]), src=r)
            elif hi > lo:
                dist.send(_r(out.contiguous()), dst=0)
        else:
            full = out
    return full, out, (lo, hi)


@dataclass
class BandOps:
    # (window, N, M) -> compact offset of every class in UC order (+ total at the end)
    slot_offsets: Callable
    # (A (N,M), window, part, nparts) -> this band's reduced sums (1-D tensor)
    compute_sums: Callable
    # (A, window, all-reduced sums, class_lo, class_hi) -> compact slots of those classes
    finalize_range: Callable
    # (full compact tensor, window, N, M, dtype, device) -> dense R
    expand_dense: Callable


def cuda_band_ops() -> BandOps:
    from .plan import Plan

    cache = {}

    def plan_for(a, window):
        key = (a.shape[0], a.shape[1], window.p, window.q, a.dtype, a.device)
        if key not in cache:
            cache[key] = Plan(a.shape[0], a.shape[1], window, dtype=a.dtype, device=a.device)
        return cache[key]

    def slot_offsets(window, n, m):
        a = torch.empty((n, m), dtype=torch.complex128, device=torch.device("cuda", torch.cuda.current_device()))
        plan = plan_for(a, window)
        return [plan.class_slot_offset(i) for i in range(plan.num_classes + 1)]

    def compute_sums(a, window, part, nparts):
        plan = plan_for(a, window)
        sums = plan.alloc_sums()
        return plan.execute_sums(a, sums, part, nparts)

    def finalize_range(a, window, sums, lo, hi):
        plan = plan_for(a, window)
        full = torch.empty(plan.output_elems("compact"), dtype=a.dtype, device=a.device)
        plan.finalize_sums(a, sums, full, "compact", lo, hi)
        return full[plan.class_slot_offset(lo):plan.class_slot_offset(hi)]

    def expand_dense(compact, window, n, m, dtype, device):
        nuc = window.p * window.q + (window.p - 1) * (window.q - 1)
        return cuda_ops().scatter_dense([compact], [list(range(nuc))], window, n, m, dtype, device)

    return BandOps(slot_offsets, compute_sums, finalize_range, expand_dense)


def class_ranges(offsets, world: int) -> list[tuple[int, int]]:
    """Contiguous class ranges with about equal slot counts (the finalize's
    work), one per rank, from the compact offsets (len = classes + 1)."""
    nc = len(offsets) - 1
    total = offsets[-1]
    bounds = [0]
    c = 0
    for r in range(1, world):
        target = total * r / world
        while c < nc and offsets[c] < target:
            c += 1
        bounds.append(max(c, bounds[-1]))
    bounds.append(nc)
    return [(bounds[r], bounds[r + 1]) for r in range(world)]


def estimate_rowband(a: torch.Tensor | None, shape: tuple[int, int], window: WindowSpec,
                     dtype=torch.complex128, device=None, gather: bool = False,
                     ops: BandOps | None = None):
    """Row-band estimate of one matrix across the process group (module
    docstring).  `a` lives on rank 0.  Returns (dense R on rank 0 if `gather`
    else None, this rank's compact slots, its class range)."""
    ops = ops or cuda_band_ops()
    rank, world = _world()
    n, m = shape
    window.validate_for(n, m)
    if device is None:
        device = a.device if (a is not None and rank == 0) else torch.device("cpu")
    buf = a if rank == 0 else torch.empty((n, m), dtype=dtype, device=device)
    if world > 1:
        dist.broadcast(_r(buf), src=0)
    sums = ops.compute_sums(buf, window, rank, world)
    if world > 1:
        dist.all_reduce(_r(sums))  # the one exchange: per-band sums -> full sums
    offsets = ops.slot_offsets(window, n, m)
    lo, hi = class_ranges(offsets, world)[rank]
    comp = ops.finalize_range(buf, window, sums, lo, hi)
    dense = None
    if gather:
        if world > 1:
            width = max(offsets[h] - offsets[l] for l, h in class_ranges(offsets, world))
            padded = torch.zeros(width, dtype=dtype, device=device)
            padded[: comp.numel()] = comp
            bucket = [torch.empty_like(padded) for _ in range(world)] if rank == 0 else None
            dist.gather(_r(padded), [_r(x) for x in bucket] if rank == 0 else None, dst=0)
            if rank == 0:
                full = torch.cat([bucket[r][: offsets[h] - offsets[l]]
                                  for r, (l, h) in enumerate(class_ranges(offsets, world))])
                dense = ops.expand_dense(full, window, n, m, dtype, device)
        else:
            dense = ops.expand_dense(comp, window, n, m, dtype, device)
    return dense, comp, (lo, hi)
