"""CPU oracle for the windowed-covariance hot path — TEST INFRASTRUCTURE ONLY.

This module restates, in plain numpy, the algorithm the reference package
``covcomb`` runs for its covariance entry point.  It is the checker the parity
tests compare the CUDA path against, and the CPU arm ``bench.py`` times.  It is
never imported by the product package (``paper_1303_2285_b200``): only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg may
load it.

Pinning: every function below is checked against golden vectors produced by
running the real reference (``tests/golden/make_golden.py`` imports ``covcomb``
from ``/root/reference/pkg/src`` in the build container and commits the
outputs under ``tests/golden/``); see ``tests/test_oracle.py``.

Conventions (0-based storage, reference ``core.py:1-11``):

* stack index k = P*cc + rr                       (``core.py:37-50``, Eq. 2.1)
* packed upper triangle, row-major                (``core.py:60-72``)
* classes (dr, dc) in the fixed UC order          (``combinations.py:53-62``)
* the reference returns the UNNORMALISED packed sum; ``covariance()`` here
  applies the 1/K normalisation that BASELINE.json's north_star asks for
  (SURVEY.md D1).
"""

from __future__ import annotations

import numpy as np

__all__ = [
    "unique_combinations",
    "packed_size",
    "packed_offset",
    "class_slot_sums",
    "class_packed_offsets",
    "estimate_packed",
    "estimate_batch_packed",
    "naive_packed",
    "dense_from_packed",
    "covariance",
    "rel_frobenius",
    "um_count",
]


def unique_combinations(p: int, q: int) -> list[tuple[int, int]]:
    """UC in the reference's order (``combinations.py:53-62``): dr in [0,p) x
    dc in [0,q) row-major, then dr in [-(p-1),-1] x dc in [1,q)."""
    out = [(dr, dc) for dr in range(p) for dc in range(q)]
    out += [(dr, dc) for dr in range(-(p - 1), 0) for dc in range(1, q)]
    return out


def packed_size(dim: int) -> int:
    return dim * (dim + 1) // 2


def packed_offset(r0: np.ndarray | int, c0: np.ndarray | int, dim: int):
    """0-based (r0 <= c0) -> packed offset; ``core.py:60-72`` shifted to 0-based."""
    return r0 * dim - (r0 * (r0 - 1)) // 2 + (c0 - r0)


def _class_pane(a: np.ndarray, dr: int, dc: int) -> np.ndarray:
    """prod[i, j] = A[i+s1, j] * conj(A[i+s2, j+dc]) (``_numba_kernels.py:80-88``).

    The (0,0) class uses re^2+im^2 so the main diagonal is exactly real, as the
    reference's numpy kernel does (``_numpy_kernels.py:34-37``).
    """
    n, m = a.shape
    if dr == 0 and dc == 0:
        return (a.real * a.real + a.imag * a.imag).astype(np.complex128)
    s1, s2 = max(-dr, 0), max(dr, 0)
    h, w = n - abs(dr), m - dc
    return a[s1:s1 + h, 0:w] * np.conj(a[s2:s2 + h, dc:dc + w])


def class_slot_sums(a: np.ndarray, dr: int, dc: int, p: int, q: int) -> np.ndarray:
    """All slot sums of one class, flat in slot order (strip u major, then v).

    Same algorithm as the reference's vectorised class kernel
    (``_numpy_kernels.py:30-53``): one product pane, a zero-padded 2-D
    inclusive prefix sum, and four-corner box sums of the fixed
    (n-p+1) x (m-q+1) box at every slot anchor (v, u).
    """
    n, m = a.shape
    prod = _class_pane(a, dr, dc)
    h, w = prod.shape
    table = np.zeros((h + 1, w + 1), dtype=np.complex128)
    np.cumsum(prod, axis=0, out=table[1:, 1:])
    np.cumsum(table[1:, 1:], axis=1, out=table[1:, 1:])
    bh, bw = n - p + 1, m - q + 1
    pv, qu = p - abs(dr), q - dc
    v = np.arange(pv)[:, None]
    u = np.arange(qu)[None, :]
    box = table[v + bh, u + bw] - table[v, u + bw] - table[v + bh, u] + table[v, u]
    return box.T.reshape(-1)


def class_packed_offsets(dr: int, dc: int, p: int, q: int) -> np.ndarray:
    """Packed offsets of a class's slots in slot order (``_numpy_kernels.py:56-64``):
    slot (u, v) sits at row k1 = p*u + s1 + v, column k1 + dc*p + dr."""
    s1 = max(-dr, 0)
    pq = p * q
    u = np.arange(q - dc)[:, None]
    v = np.arange(p - abs(dr))[None, :]
    k1 = (p * u + s1 + v).reshape(-1)
    return packed_offset(k1, k1 + dc * p + dr, pq)


def _as_c128(a) -> np.ndarray:
    arr = np.array(a, dtype=np.complex128, order="C")  # core.py:101-108 coercion
    if arr.ndim != 2 or arr.shape[0] < 1 or arr.shape[1] < 1:
        raise ValueError(f"input matrix must be 2-D and non-empty, got {arr.shape}")
    return arr


def estimate_packed(a, p: int, q: int, classes=None) -> np.ndarray:
    """Unnormalised packed upper triangle, class decomposition
    (``engine.py:108-147`` driving ``_numpy_kernels.apply_combination``).

    ``classes`` optionally restricts the computation to a subset of UC (the
    remaining packed slots stay zero) — used to spot-check large configs."""
    arr = _as_c128(a)
    n, m = arr.shape
    if p < 1 or q < 1 or p > n or q > m:
        raise ValueError(f"{p}x{q} window does not fit a {n}x{m} matrix")
    out = np.zeros(packed_size(p * q), dtype=np.complex128)
    for dr, dc in (unique_combinations(p, q) if classes is None else classes):
        out[class_packed_offsets(dr, dc, p, q)] = class_slot_sums(arr, dr, dc, p, q)
    return out


def estimate_batch_packed(stack, p: int, q: int) -> list[np.ndarray]:
    """Per-snapshot packed results (``engine.py:219-255``)."""
    return [estimate_packed(x, p, q) for x in stack]


def naive_packed(a, p: int, q: int) -> np.ndarray:
    """Direct Eq. (2.2) sweep (``baseline.py:35-46``, ``_numba_kernels.py:14-32``):
    every placement's column-stacked vector v adds v v^H to the upper triangle.
    Pure numpy per placement — small cases only."""
    arr = _as_c128(a)
    n, m = arr.shape
    pq = p * q
    rows, cols = np.triu_indices(pq)
    diag = rows == cols
    out = np.zeros(packed_size(pq), dtype=np.complex128)
    for wr in range(n - p + 1):
        for wc in range(m - q + 1):
            v = arr[wr:wr + p, wc:wc + q].ravel(order="F")  # k = p*cc + rr
            prod = v[rows] * np.conj(v[cols])
            prod[diag] = (v.real * v.real + v.imag * v.imag)[rows[diag]]
            out += prod
    return out


def dense_from_packed(packed: np.ndarray, dim: int) -> np.ndarray:
    """Hermitian dense matrix from the packed triangle (``core.py:170-176``):
    lower = conj(upper); the stored diagonal is kept as is."""
    r, c = np.triu_indices(dim)
    out = np.empty((dim, dim), dtype=np.complex128)
    out[c, r] = np.conj(packed)
    out[r, c] = packed
    return out


def covariance(a, p: int, q: int) -> np.ndarray:
    """Dense normalised R = (1/K) sum x x^H — the north_star's output."""
    arr = _as_c128(a)
    n, m = arr.shape
    k = (n - p + 1) * (m - q + 1)
    return dense_from_packed(estimate_packed(arr, p, q), p * q) / k


def rel_frobenius(a, b) -> float:
    """||a-b||_F / ||b||_F, 0 when both vanish (``core.py:179-186``)."""
    a = np.asarray(a)
    b = np.asarray(b)
    den = float(np.linalg.norm(b))
    if den == 0.0:
        return 0.0 if float(np.linalg.norm(a)) == 0.0 else float("inf")
    return float(np.linalg.norm(a - b)) / den


def um_count(n: int, m: int, p: int, q: int) -> int:
    """Unique complex products (``analysis.py:46-56``, Eq. 4.6)."""
    um1 = (p * (2 * n - p + 1) // 2) * (q * (2 * m - q + 1) // 2)
    um2 = ((p - 1) * (2 * n - p) // 2) * ((q - 1) * (2 * m - q) // 2)
    return um1 + um2
