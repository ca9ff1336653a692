"""GPU naive estimator: the direct Eq. (2.2) definition the
reference's ``baseline.estimate_naive`` sweeps (``baseline.py:35-46``),
R = (1/K) X X^H with X[k, w] = A[wr+rr, wc+cc], k = P*cc + rr, evaluated as a
chunked implicit-im2col Gram product on the tensor cores (cuBLAS ZGEMM /
CGEMM through torch).  It shares no code or algorithm with the class kernels,
so it is the independent cross-check behind ``verify`` (cli.py); it costs
8*K*PQ(PQ+1)/2-ish flops (about 1000x the class decomposition at cfg5).
"""

from __future__ import annotations

import torch

from .core import WindowSpec, _to_device_matrix

__all__ = ["estimate_naive"]


def _windows(a: torch.Tensor, p: int, q: int) -> torch.Tensor:
    # (wr, wc, rr, cc) -> rows k = p*cc + rr, columns = placements
    t = a.unfold(0, p, 1).unfold(1, q, 1).permute(3, 2, 0, 1)
    return t.reshape(p * q, -1)


@torch.no_grad()
def estimate_naive(a, window: WindowSpec, device=None, chunk_bytes: int = 1 << 30) -> torch.Tensor:
    """Dense normalised R on the GPU by the window-sum definition."""
    t = _to_device_matrix(a, device, None, ndim=2)
    n, m = t.shape
    window.validate_for(n, m)
    p, q = window.p, window.q
    bh, bw = n - p + 1, m - q + 1
    per_row = p * q * bw * t.element_size()
    rows = max(1, min(bh, chunk_bytes // max(per_row, 1)))
    acc = torch.zeros((p * q, p * q), dtype=t.dtype, device=t.device)
    for w0 in range(0, bh, rows):
        x = _windows(t[w0:w0 + min(rows, bh - w0) + p - 1], p, q)
        acc += x @ x.conj().T
    return acc / (bh * bw)
