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

* ``estimate_rowband`` — the single large estimate on the spectral (or
  tensor-core) path: the sums the kernels accumulate (CC, edge-column and
  edge-row sums) are sums over A's rows, so they split into a FIXED number of
  row parts (``ROWBAND_PARTS``, independent of the GPU count); each rank
  computes a contiguous run of parts (``covgpu_plan_execute_sums``), and ONE
  all-to-all sends every rank exactly the slices of each part that its
  finalize range needs (``covgpu_plan_sums_range``; a reduce-scatter with a
  fixed order).  Each rank adds the parts in part order and finalizes a
  contiguous, slot-balanced range of classes (``covgpu_plan_finalize_sums``),
  so R is bitwise identical on 1, 2, 4 or 8 GPUs.  A rank needs only the
  rows its parts read (``covgpu_plan_band_rows``) plus the strips: A can be
  distributed by row bands instead of broadcast (``rowband_regions``).
  Rank 0 gathers the compact ranges on request.

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
           "BandOps", "cuda_band_ops", "estimate_rowband", "class_ranges", "part_ranges", "rowband_regions",
           "simulate_rowband", "ROWBAND_PARTS"]


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


def _resolve_device(a, rank: int, device, cuda_default: bool) -> torch.device:
    """The device of this rank's buffers: the given one, rank 0's input's,
    else the current CUDA device for the CUDA ops (CPU only for injected
    test ops)."""
    if device is not None:
        return torch.device(device)
    if a is not None and rank == 0:
        return a.device
    if cuda_default and torch.cuda.is_available():
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


_DTYPE_CODE = {torch.complex128: 0, torch.complex64: 1}


def _check_root_input(buf: torch.Tensor, dtype, rank: int, world: int) -> None:
    """Rank 0's input must match what the other ranks allocated (dtype,
    shape, contiguity): its description is broadcast and checked on every
    rank before the data broadcast (a mismatch would corrupt or hang it)."""
    if rank == 0 and (buf.dtype not in _DTYPE_CODE or not buf.is_contiguous()):
        raise ValueError("rank 0's input must be a contiguous complex64 / complex128 tensor")
    if world == 1:
        return
    desc = torch.tensor([_DTYPE_CODE.get(buf.dtype, -1), *buf.shape] if rank == 0 else [0] * (1 + buf.dim()),
                        dtype=torch.int64, device=buf.device)
    dist.broadcast(desc, src=0)
    want = [_DTYPE_CODE[dtype], *buf.shape] if rank != 0 else desc.tolist()
    ok = torch.tensor([1 if desc.tolist() == want else 0], dtype=torch.int64, device=buf.device)
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)  # every rank refuses together
    if not int(ok.item()):
        raise ValueError(f"rank 0's input (dtype code, shape) {desc.tolist()} does not match what the "
                         f"other ranks expect")


def estimate_sharded(a: torch.Tensor | None, shape: tuple[int, int], window: WindowSpec,
                     dtype=torch.complex128, device=None, gather: bool = False,
                     ops: ShardOps | None = None):
    """Class-sharded estimate of one matrix across the process group.

    `a` is the (N, M) input on rank 0 (ignored elsewhere).  Returns
    (dense R on rank 0 if `gather` else None, this rank's compact shard,
    this rank's class ids)."""
    cuda_default = ops is None
    ops = ops or cuda_ops()
    rank, world = _world()
    n, m = shape
    window.validate_for(n, m)
    device = _resolve_device(a, rank, device, cuda_default)
    buf = a if rank == 0 else torch.empty((n, m), dtype=dtype, device=device)
    _check_root_input(buf, dtype, rank, world)
    dtype = buf.dtype
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
    cuda_default = ops is None
    ops = ops or cuda_ops()
    rank, world = _world()
    batch, n, m = shape
    window.validate_for(n, m)
    device = _resolve_device(stack, rank, device, cuda_default)
    if rank == 0 and (stack.dtype != dtype or tuple(stack.shape) != (batch, n, m)):
        raise ValueError(f"rank 0's stack {stack.dtype} {tuple(stack.shape)} does not match {dtype} {shape}")
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


ROWBAND_PARTS = 8  # fixed row-part count of the row-band mode (any GPU count gives the same bits)


@dataclass
class BandOps:
    # (A, window) -> compact offset of every plan class (+ total at the end)
    slot_offsets: Callable
    # (A (N,M), window, part, nparts) -> this part's sums (1-D complex tensor)
    compute_sums: Callable
    # (A, window, class_lo, class_hi) -> [(begin, end), ...] sums-buffer slices of those classes
    sums_slices: Callable
    # (A, window, sums holding at least the range's slices, class_lo, class_hi) -> compact slots
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

    def slot_offsets(a, window):
        plan = plan_for(a, window)
        return [plan.class_slot_offset(i) for i in range(plan.num_classes + 1)]

    def compute_sums(a, window, part, nparts):
        plan = plan_for(a, window)
        sums = plan.alloc_sums()
        return plan.execute_sums(a, sums, part, nparts)

    def sums_slices(a, window, lo, hi):
        return plan_for(a, window).sums_range(lo, hi)

    def finalize_range(a, window, sums, lo, hi):
        plan = plan_for(a, window)
        full = torch.empty(plan.output_elems("compact"), dtype=a.dtype, device=a.device)
        plan.finalize_sums(a, sums, full, "compact", lo, hi)
        return full[plan.class_slot_offset(lo):plan.class_slot_offset(hi)]

    def expand_dense(compact, window, n, m, dtype, device):
        nuc = window.p * window.q + (window.p - 1) * (window.q - 1)
        return cuda_ops().scatter_dense([compact], [list(range(nuc))], window, n, m, dtype, device)

    return BandOps(slot_offsets, compute_sums, sums_slices, finalize_range, expand_dense)


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


def part_ranges(nparts: int, world: int) -> list[tuple[int, int]]:
    """Contiguous runs of row parts per rank (part order = rank order)."""
    return [(nparts * r // world, nparts * (r + 1) // world) for r in range(world)]


def rowband_regions(plan, parts: tuple[int, int], nparts: int = ROWBAND_PARTS):
    """The regions of A a rank running row parts [parts[0], parts[1]) reads:
    [(row_begin, row_end, col_begin, col_end), ...] — its band rows (all
    columns), the top / bottom P-1 strip rows and the first / last Q-1
    columns of every row (covgpu_plan_band_rows)."""
    n, m, p, q = plan.n, plan.m, plan.window.p, plan.window.q
    regs = []
    for part in range(*parts):
        r0, r1 = plan.band_rows(part, nparts)
        regs.append((r0, r1, 0, m))
    regs += [(0, p - 1, 0, m), (n - p + 1, n, 0, m), (0, n, 0, q - 1), (0, n, m - q + 1, m)]
    return [r for r in regs if r[1] > r[0] and r[3] > r[2]]


def _all_to_all(send: list[torch.Tensor], recv_sizes: list[int], like: torch.Tensor) -> list[torch.Tensor]:
    """One all-to-all of variable-size complex chunks (world >= 1)."""
    rank, world = _world()
    if world == 1:
        return [send[0]]
    out = torch.empty(sum(recv_sizes), dtype=like.dtype, device=like.device)
    inp = torch.cat(send) if send else torch.empty(0, dtype=like.dtype, device=like.device)
    in_sz = [int(t.numel()) for t in send]
    dist.all_to_all_single(_r(out), _r(inp), output_split_sizes=recv_sizes, input_split_sizes=in_sz)
    return list(torch.split(out, recv_sizes))


def _rowband_send(parts: list[torch.Tensor], slices: list[list[tuple[int, int]]]) -> list[torch.Tensor]:
    """Chunks for every destination q: for each of the sender's parts
    (ascending), the slices of q's class range."""
    out = []
    for sl in slices:
        chunks = [part[b:e] for part in parts for b, e in sl]
        out.append(torch.cat(chunks) if chunks else parts[0][:0])
    return out


def _rowband_reduce(received: list[torch.Tensor], width: int, slices: list[tuple[int, int]],
                    like: torch.Tensor) -> torch.Tensor:
    """Sums buffer holding this rank's class range: the parts' slices added
    in part order (sources ascending, each sending its parts ascending)."""
    mine = [c for chunk in received for c in torch.split(chunk, width)] if width else []
    sums = torch.zeros_like(like)
    if mine:
        total = mine[0].clone()
        for c in mine[1:]:
            total += c
        pos = 0
        for b, e in slices:
            sums[b:e] = total[pos:pos + (e - b)]
            pos += e - b
    return sums


def estimate_rowband(a: torch.Tensor | None, shape: tuple[int, int], window: WindowSpec,
                     dtype=torch.complex128, device=None, gather: bool = False,
                     ops: BandOps | None = None, nparts: int = ROWBAND_PARTS, distribute: str = "broadcast"):
    """Row-band estimate of one matrix across the process group (module
    docstring).  distribute="broadcast": `a` lives on rank 0 and is
    broadcast; "local": every rank passes its own (N, M) buffer holding at
    least ``rowband_regions`` of its parts.  Returns (dense R on rank 0 if
    `gather` else None, this rank's compact slots, its class range)."""
    cuda_default = ops is None
    ops = ops or cuda_band_ops()
    rank, world = _world()
    n, m = shape
    window.validate_for(n, m)
    if world > nparts:
        raise ValueError(f"{world} ranks need at least as many row parts (nparts={nparts})")
    device = _resolve_device(a, rank, device, cuda_default)
    if distribute == "local":
        if a is None or tuple(a.shape) != (n, m):
            raise ValueError("distribute='local' needs every rank's (N, M) buffer")
        buf = a
    else:
        buf = a if rank == 0 else torch.empty((n, m), dtype=dtype, device=device)
        _check_root_input(buf, dtype, rank, world)
        if world > 1:
            dist.broadcast(_r(buf), src=0)
    p_lo, p_hi = part_ranges(nparts, world)[rank]
    parts = [ops.compute_sums(buf, window, part, nparts) for part in range(p_lo, p_hi)]
    offsets = ops.slot_offsets(buf, window)
    ranges = class_ranges(offsets, world)
    slices = [ops.sums_slices(buf, window, lo_q, hi_q) for lo_q, hi_q in ranges]
    width = [sum(e - b for b, e in sl) for sl in slices]
    send = _rowband_send(parts, slices)
    recv_sizes = [(hi - lo) * width[rank] for lo, hi in part_ranges(nparts, world)]
    got = _all_to_all(send, recv_sizes, parts[0])
    sums = _rowband_reduce(got, width[rank], slices[rank], parts[0])
    lo, hi = ranges[rank]
    comp = ops.finalize_range(buf, window, sums, lo, hi)
    dense = None
    if gather:
        if world > 1:
            wmax = max(offsets[h] - offsets[l] for l, h in ranges)
            padded = torch.zeros(wmax, dtype=comp.dtype, device=comp.device)
            padded[: comp.numel()] = comp
            bucket = [torch.empty_like(padded) for _ in range(world)] if rank == 0 else None
            dist.gather(_r(padded), [_r(x) for x in bucket] if rank == 0 else None, dst=0)
            if rank == 0:
                full = torch.cat([bucket[r][: offsets[h] - offsets[l]] for r, (l, h) in enumerate(ranges)])
                dense = ops.expand_dense(full, window, n, m, comp.dtype, comp.device)
        else:
            dense = ops.expand_dense(comp, window, n, m, comp.dtype, comp.device)
    return dense, comp, (lo, hi)


def simulate_rowband(bufs: list[torch.Tensor], window: WindowSpec, ops: BandOps | None = None,
                     nparts: int = ROWBAND_PARTS) -> torch.Tensor:
    """The row-band estimate of `len(bufs)` ranks run one after another in
    this process (rank r on bufs[r]; the all-to-all and the gather become
    list routing): the same computation, per rank and per part, as
    estimate_rowband on that many GPUs — for testing N-invariance on one
    device.  Returns the dense R rank 0 would assemble."""
    ops = ops or cuda_band_ops()
    world = len(bufs)
    n, m = bufs[0].shape
    offsets = ops.slot_offsets(bufs[0], window)
    ranges = class_ranges(offsets, world)
    slices = [ops.sums_slices(bufs[0], window, lo, hi) for lo, hi in ranges]
    width = [sum(e - b for b, e in sl) for sl in slices]
    sends = []
    for r in range(world):
        p_lo, p_hi = part_ranges(nparts, world)[r]
        parts = [ops.compute_sums(bufs[r], window, part, nparts) for part in range(p_lo, p_hi)]
        sends.append((_rowband_send(parts, slices), parts[0]))
    comps = []
    for q in range(world):
        sums = _rowband_reduce([sends[p][0][q] for p in range(world)], width[q], slices[q], sends[0][1])
        comps.append(ops.finalize_range(bufs[q], window, sums, *ranges[q]))
    return ops.expand_dense(torch.cat(comps), window, n, m, comps[0].dtype, comps[0].device)
