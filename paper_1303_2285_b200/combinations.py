"""Offset classes (the work decomposition), host-side integer logic.

Mirrors the reference's ``combinations`` module (``combinations.py:53-85``):
the unique-combination set UC in its fixed order, the per-class product count
mu and slot count eta, the output diagonal, and the bulk-kernel work groups
(consecutive row lags of one column lag) that the GPU kernels and the
partitioner operate on.
"""

from __future__ import annotations

from dataclasses import dataclass

from .core import WindowSpec

__all__ = [
    "Combination",
    "unique_combinations",
    "is_unique_combination",
    "class_index",
    "pair_count",
    "max_writes",
    "lag_group_size",
    "work_groups",
    "um_count",
]


@dataclass(frozen=True)
class Combination:
    """Inter-element offset (dr, dc) naming one independent unit of work."""

    dr: int
    dc: int

    def diag_offset(self, p: int) -> int:
        """Output diagonal the class writes: col - row = dc*p + dr
        (``combinations.py:41-43``)."""
        return self.dc * p + self.dr


def unique_combinations(window: WindowSpec) -> list[Combination]:
    """UC in the reference's order (``combinations.py:53-62``)."""
    p, q = window.p, window.q
    first = [Combination(dr, dc) for dr in range(p) for dc in range(q)]
    second = [Combination(dr, dc) for dr in range(-(p - 1), 0) for dc in range(1, q)]
    return first + second


def is_unique_combination(dr: int, dc: int, window: WindowSpec) -> bool:
    if 0 <= dr <= window.p - 1 and 0 <= dc <= window.q - 1:
        return True
    return -(window.p - 1) <= dr <= -1 and 1 <= dc <= window.q - 1


def class_index(dr: int, dc: int, window: WindowSpec) -> int:
    """Position of (dr, dc) in UC order (inverse of ``unique_combinations``)."""
    p, q = window.p, window.q
    if not is_unique_combination(dr, dc, window):
        raise ValueError(f"offset ({dr}, {dc}) is not a unique combination for a {p}x{q} window")
    return dr * q + dc if dr >= 0 else p * q + (dr + p - 1) * (q - 1) + (dc - 1)


def pair_count(comb: Combination, n: int, m: int) -> int:
    """mu = (n-|dr|)(m-|dc|) products of the class (``combinations.py:71-77``)."""
    return (n - abs(comb.dr)) * (m - abs(comb.dc))


def max_writes(comb: Combination, window: WindowSpec) -> int:
    """eta = (p-|dr|)(q-|dc|) slots owned by the class (``combinations.py:80-85``)."""
    if abs(comb.dr) >= window.p or abs(comb.dc) >= window.q:
        raise ValueError(
            f"offset ({comb.dr}, {comb.dc}) does not fit a {window.p}x{window.q} window"
        )
    return (window.p - abs(comb.dr)) * (window.q - abs(comb.dc))


def lag_group_size(p: int) -> int:
    """Row lags E one bulk warp carries in its register window (covgpu.cu pick_E)."""
    span = 2 * p - 1
    return 4 if span <= 4 else 8 if span <= 8 else 16


def work_groups(window: WindowSpec) -> list[tuple[int, int, list[int]]]:
    """Bulk-kernel work groups in launch order: (dc, dr0, [UC indices]).

    A group is E consecutive row lags dr0..dr0+E-1 of one column lag dc; the
    lags outside UC are dropped.  Must match covgpu.cu covgpu_plan_create.
    """
    p, q = window.p, window.q
    e = lag_group_size(p)
    out = []
    for dc in range(q):
        first = 0 if dc == 0 else -(p - 1)
        for dr0 in range(first, p, e):
            ids = [class_index(dr, dc, window) for dr in range(dr0, min(dr0 + e, p))]
            out.append((dc, dr0, ids))
    return out


def um_count(n: int, m: int, p: int, q: int) -> int:
    """Unique complex products UM = UM1 + UM2 (``analysis.py:46-56``, Eq. 4.6)."""
    um1 = (p * (2 * n - p + 1) // 2) * (q * (2 * m - q + 1) // 2)
    um2 = ((p - 1) * (2 * n - p) // 2) * ((q - 1) * (2 * m - q) // 2)
    return um1 + um2
