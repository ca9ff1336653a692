"""Work partitioner: balance offset classes across GPUs (and launches).

The unit is a bulk work group (E consecutive row lags of one column lag,
``combinations.work_groups``), so every class is computed by the same warps
with the same reduction order whatever the shard count — results are
bitwise identical for 1..G shards.  Cost per group is the
products it forms, sum of mu = (N-|dr|)(M-dc) over its classes, which replaces
the reference's modelled dispatch cost mu*(1+eta) (``engine.py:86-92``); the
split is static, deterministic and contiguous in the canonical group order.
"""

from __future__ import annotations

from .combinations import Combination, pair_count, unique_combinations, work_groups
from .core import WindowSpec

__all__ = ["group_costs", "partition_classes", "shard_cost"]


def group_costs(n: int, m: int, window: WindowSpec):
    """[(ids, cost)] per work group in canonical order."""
    combos = unique_combinations(window)
    out = []
    for _dc, _dr0, ids in work_groups(window):
        out.append((ids, sum(pair_count(combos[i], n, m) for i in ids)))
    return out


def partition_classes(n: int, m: int, window: WindowSpec, shards: int) -> list[list[int]]:
    """Split UC into `shards` lists of class ids with near-equal product counts.

    Contiguous greedy over the canonical group order: shard s closes once the
    running cost reaches (s+1)/shards of the total.  Shards may be empty when
    there are fewer groups than shards.
    """
    if shards < 1:
        raise ValueError(f"shards must be >= 1, got {shards}")
    groups = group_costs(n, m, window)
    total = sum(c for _, c in groups)
    out: list[list[int]] = [[] for _ in range(shards)]
    run = 0
    s = 0
    for ids, cost in groups:
        # move on when this shard already holds its share
        while s < shards - 1 and run >= total * (s + 1) / shards:
            s += 1
        out[s].extend(ids)
        run += cost
    return out


def shard_cost(n: int, m: int, window: WindowSpec, ids) -> int:
    combos = unique_combinations(window)
    return sum(pair_count(combos[i], n, m) for i in ids)
