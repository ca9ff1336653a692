"""Boundary types: window, input matrix, covariance result.

Index conventions follow the reference (``core.py:1-11``): logical indices are
1-based at the accessors, storage is 0-based; the stacked index of window
element (rr, cc) is k = P*cc + rr (Eq. 2.1, ``core.py:37-50``).

Differences from the reference, all required by BASELINE.json's north_star:
* the result lives on the GPU as a dense, exactly Hermitian PQ x PQ tensor
  normalised by 1/K; ``.packed`` gives the reference's packed upper triangle
  (``core.py:140-176``) of that normalised matrix;
* complex64 inputs stay complex64 (FP32 path); every other input is coerced to
  complex128 like the reference (``core.py:101-108``).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

__all__ = [
    "MAX_PACKED_ENTRIES",
    "WindowSpec",
    "InputMatrix",
    "CovarianceMatrix",
    "as_input_matrix",
    "column_stack_index",
    "packed_offset",
    "packed_size",
    "rel_frobenius_distance",
    "max_rel_diff",
]

MAX_PACKED_ENTRIES = 2**31 - 1  # core.py:34


def column_stack_index(r_rel: int, c_rel: int, p: int, q: int | None = None) -> int:
    """1-based stack position of window element (r_rel, c_rel) (``core.py:37-50``)."""
    if p < 1:
        raise IndexError(f"window height must be >= 1, got {p}")
    if not 1 <= r_rel <= p:
        raise IndexError(f"relative row {r_rel} outside window of height {p}")
    if c_rel < 1 or (q is not None and c_rel > q):
        raise IndexError(f"relative column {c_rel} outside window of width {q}")
    return p * (c_rel - 1) + r_rel


def packed_size(dim: int) -> int:
    if dim < 1:
        raise ValueError(f"matrix dimension must be >= 1, got {dim}")
    return dim * (dim + 1) // 2


def packed_offset(r: int, c: int, dim: int) -> int:
    """0-based packed offset of 1-based upper-triangle entry (r, c) (``core.py:60-72``)."""
    if r < 1 or c > dim:
        raise IndexError(f"({r}, {c}) outside a {dim}x{dim} matrix")
    if r > c:
        raise ValueError(f"({r}, {c}) lies in the lower triangle; read ({c}, {r}) and conjugate")
    return (r - 1) * dim - (r - 1) * (r - 2) // 2 + (c - r)


@dataclass(frozen=True)
class WindowSpec:
    """Sliding window dimensions: height p, width q (``core.py:75-93``)."""

    p: int
    q: int

    def __post_init__(self) -> None:
        if self.p < 1 or self.q < 1:
            raise ValueError(f"window dimensions must be positive, got {self.p}x{self.q}")

    @property
    def stack_size(self) -> int:
        return self.p * self.q

    def validate_for(self, n: int, m: int) -> None:
        if self.p > n or self.q > m:
            raise ValueError(f"{self.p}x{self.q} window does not fit a {n}x{m} matrix")


_COMPLEX_TORCH = {torch.complex128: np.complex128, torch.complex64: np.complex64}


class InputMatrix:
    """Dense complex N x M signal matrix on the GPU (immutable by contract).

    Accepts anything the reference accepts (nested lists, numpy arrays, real
    or complex) plus torch tensors.  complex64 data stays complex64; all other
    data is coerced to complex128 (``core.py:101-108``).
    """

    __slots__ = ("tensor",)

    def __init__(self, values, device=None, dtype=None) -> None:
        self.tensor = _to_device_matrix(values, device, dtype, ndim=2)

    @property
    def n(self) -> int:
        return self.tensor.shape[0]

    @property
    def m(self) -> int:
        return self.tensor.shape[1]

    @property
    def dtype(self) -> torch.dtype:
        return self.tensor.dtype

    @property
    def array(self) -> np.ndarray:
        return self.tensor.cpu().numpy()

    def at(self, r: int, c: int) -> complex:
        if not (1 <= r <= self.n and 1 <= c <= self.m):
            raise IndexError(f"({r}, {c}) outside a {self.n}x{self.m} matrix")
        return complex(self.tensor[r - 1, c - 1].item())

    @classmethod
    def random(cls, n: int, m: int, seed, device=None) -> "InputMatrix":
        """Re and im uniform in [-1, 1), PCG64 — the reference's generator
        (``core.py:124-132``), so a seed gives the same matrix as there."""
        rng = np.random.default_rng(seed)
        return cls(rng.uniform(-1.0, 1.0, (n, m)) + 1j * rng.uniform(-1.0, 1.0, (n, m)), device)


def _default_device(device):
    if device is not None:
        return torch.device(device)
    if not torch.cuda.is_available():
        raise RuntimeError("covgpu needs a CUDA device (there is no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _to_device_matrix(values, device, dtype, ndim: int) -> torch.Tensor:
    if isinstance(values, InputMatrix):
        values = values.tensor
    if isinstance(values, torch.Tensor):
        t = values
        if dtype is None:
            dtype = torch.complex64 if t.dtype == torch.complex64 else torch.complex128
        dev = torch.device(device) if device is not None else (
            t.device if t.is_cuda else _default_device(None))
        t = t.to(device=dev, dtype=dtype).contiguous()
    else:
        arr = np.asarray(values)
        if dtype is None:
            dtype = torch.complex64 if arr.dtype == np.complex64 else torch.complex128
        npdt = np.complex64 if dtype == torch.complex64 else np.complex128
        arr = np.array(values, dtype=npdt, order="C")
        t = torch.from_numpy(arr).to(_default_device(device))
    if dtype not in (torch.complex128, torch.complex64):
        raise ValueError(f"unsupported dtype {dtype}; expected complex128 or complex64")
    if t.dim() != ndim:
        raise ValueError(f"input matrix must be {ndim}-D, got shape {tuple(t.shape)}")
    if any(s < 1 for s in t.shape):
        raise ValueError(f"input matrix must be non-empty, got shape {tuple(t.shape)}")
    return t


def as_input_matrix(values, device=None) -> InputMatrix:
    return values if isinstance(values, InputMatrix) else InputMatrix(values, device)


class CovarianceMatrix:
    """Normalised Hermitian estimate R = (1/K) sum x x^H, dense on the GPU.

    ``dense()`` returns the device tensor; ``packed`` the reference's packed
    upper triangle (``core.py:140-162``) of R; ``at(r, c)`` resolves 1-based
    entries like the reference (``core.py:164-168``).  ``k`` is the number of
    window placements; ``k * R`` is the reference's unnormalised sum.
    """

    __slots__ = ("dim", "k", "_dense")

    def __init__(self, dense: torch.Tensor, k: int) -> None:
        size = packed_size(dense.shape[-1])
        if size > MAX_PACKED_ENTRIES:
            raise ValueError(
                f"packed triangle of a {dense.shape[-1]}x{dense.shape[-1]} matrix needs {size} "
                f"entries, beyond the {MAX_PACKED_ENTRIES} capacity"
            )
        self.dim = dense.shape[-1]
        self.k = k
        self._dense = dense

    def dense(self) -> torch.Tensor:
        return self._dense

    @property
    def packed(self) -> torch.Tensor:
        r, c = torch.triu_indices(self.dim, self.dim, device=self._dense.device)
        return self._dense[r, c]

    def at(self, r: int, c: int) -> complex:
        if not (1 <= r <= self.dim and 1 <= c <= self.dim):
            raise IndexError(f"({r}, {c}) outside a {self.dim}x{self.dim} matrix")
        return complex(self._dense[r - 1, c - 1].item())

    def numpy(self) -> np.ndarray:
        return self._dense.cpu().numpy()


def rel_frobenius_distance(a, b) -> float:
    """||a - b|| / ||b||; 0 when both are zero (``core.py:179-186``)."""
    a = a.cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a)
    b = b.cpu().numpy() if isinstance(b, torch.Tensor) else np.asarray(b)
    denom = float(np.linalg.norm(b))
    if denom == 0.0:
        return 0.0 if float(np.linalg.norm(a)) == 0.0 else float("inf")
    return float(np.linalg.norm(a.astype(np.complex128) - b.astype(np.complex128))) / denom


def max_rel_diff(a, b) -> float:
    """Largest entry difference relative to the larger max modulus (``core.py:189-196``)."""
    a = a.cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a)
    b = b.cpu().numpy() if isinstance(b, torch.Tensor) else np.asarray(b)
    scale = max(float(np.abs(a).max(initial=0.0)), float(np.abs(b).max(initial=0.0)))
    if scale == 0.0:
        return 0.0
    return float(np.abs(a.astype(np.complex128) - b.astype(np.complex128)).max(initial=0.0)) / scale
