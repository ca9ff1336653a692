"""Work partitioner: balance offset classes across GPUs.

The unit is one bulk-kernel CTA column of work: `lags` consecutive row lags
(dr) x `warps` consecutive column lags (dc) — all classes that share one walk
over A's rows (``csrc/bulk.cuh``).  A shard made of whole units launches no
partially used CTAs.  Unit cost = products formed, sum of
mu = (N-|dr|)(M-dc) over its classes (``combinations.py:71-77``), replacing
the reference's modelled dispatch cost mu*(1+eta) (``engine.py:86-92``).
Units are assigned longest-first to the least-loaded shard (LPT, the policy
of the reference's scheduling simulator, ``schedsim.py:116-131``) —
deterministic, so every rank computes the same partition.  A class's result
does not depend on which shard computes it (no shared reductions), so any
partition reproduces the unsharded result bit for bit.
"""

from __future__ import annotations

import heapq

from .combinations import class_index, is_unique_combination, pair_count, unique_combinations
from .core import WindowSpec

__all__ = ["bulk_geometry", "work_units", "partition_classes", "shard_cost"]


def bulk_geometry(p: int, fp64: bool = True, n: int = 2048, m: int = 2048, q: int = 64,
                  batch: int = 1) -> tuple[int, int]:
    """(row lags, column lags) per bulk CTA — mirrors covgpu.cu pick_bulk_variant
    (checked against covgpu_bulk_geometry in tests)."""
    span = 2 * p - 1

    def waves(e, nw, minb):
        ctas = batch * ((span + e - 1) // e) * ((q + nw - 1) // nw) * ((m + 31) // 32)
        return ctas / (148.0 * minb)

    if span <= 4:
        return 4, 8
    if fp64:
        return (16, 4) if span > 8 and waves(16, 4, 2) >= 6.0 else (8, 4)
    return (8, 8) if waves(8, 8, 2) >= 6.0 else (8, 4)


def work_units(n: int, m: int, window: WindowSpec, fp64: bool = True):
    """[(class ids, cost)] per bulk unit in launch order."""
    p, q = window.p, window.q
    lags, warps = bulk_geometry(p, fp64, n, m, q)
    units = []
    for drg in range((2 * p - 1 + lags - 1) // lags):
        dr0 = -(p - 1) + drg * lags
        for dcb in range((q + warps - 1) // warps):
            ids = []
            for dr in range(dr0, min(dr0 + lags, p)):
                for dc in range(dcb * warps, min((dcb + 1) * warps, q)):
                    if is_unique_combination(dr, dc, window):
                        ids.append(class_index(dr, dc, window))
            if ids:
                units.append((sorted(ids), sum((n - abs(_dr(i, p, q))) * (m - _dc(i, p, q))
                                                 for i in ids)))
    return units


def _dr(i: int, p: int, q: int) -> int:
    return i // q if i < p * q else (i - p * q) // (q - 1) - (p - 1)


def _dc(i: int, p: int, q: int) -> int:
    return i % q if i < p * q else (i - p * q) % (q - 1) + 1


def partition_classes(n: int, m: int, window: WindowSpec, shards: int,
                      fp64: bool = True) -> list[list[int]]:
    """Split UC into `shards` sorted lists of class ids (LPT over bulk units)."""
    if shards < 1:
        raise ValueError(f"shards must be >= 1, got {shards}")
    units = work_units(n, m, window, fp64)
    order = sorted(range(len(units)), key=lambda u: (-units[u][1], u))
    heap = [(0, s) for s in range(shards)]
    out: list[list[int]] = [[] for _ in range(shards)]
    for u in order:
        load, s = heapq.heappop(heap)
        out[s].extend(units[u][0])
        heapq.heappush(heap, (load + units[u][1], s))
    return [sorted(s) for s in out]


def shard_cost(n: int, m: int, window: WindowSpec, ids) -> int:
    combos = unique_combinations(window)
    return sum(pair_count(combos[i], n, m) for i in ids)
