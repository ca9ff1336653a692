"""GPU naive cross-check — TEST INFRASTRUCTURE ONLY.

An independent, mostly GPU-side oracle for sizes where the CPU oracle is slow
(cfg5: ~20 min in numpy): the direct Eq. (2.2) definition the reference's
baseline sweeps (``baseline.py:35-46``),

    R = (1/K) X X^H,   X[k, w] = A[wr + rr, wc + cc],  k = P*cc + rr,

evaluated as a chunked implicit-im2col Gram product with cuBLAS (ZGEMM /
CGEMM through torch).  It shares nothing with the covgpu kernels (no classes,
no recurrence), so agreement is meaningful; its own rounding is that of a
plain sum over K placements in blocks.
"""

from __future__ import annotations

import torch


def _window_matrix(a: torch.Tensor, p: int, q: int) -> torch.Tensor:
    """(PQ, n_windows) with rows in column-stack order k = p*cc + rr."""
    n, m = a.shape
    # unfold rows then columns: (n-p+1, m-q+1, p, q) -> rows k = p*cc + rr
    t = a.unfold(0, p, 1).unfold(1, q, 1)  # (wr, wc, rr, cc)
    t = t.permute(3, 2, 0, 1)  # (cc, rr, wr, wc)
    return t.reshape(p * q, -1)


@torch.no_grad()
def covariance_gram(a: torch.Tensor, p: int, q: int, rows_per_chunk: int | None = None,
                    accum_dtype: torch.dtype = torch.complex128) -> torch.Tensor:
    """Dense normalised R on a's device, by chunks of window rows."""
    n, m = a.shape
    bh, bw = n - p + 1, m - q + 1
    pq = p * q
    if rows_per_chunk is None:
        # keep each X chunk around 1 GiB
        per_row = pq * bw * torch.empty((), dtype=accum_dtype).element_size()
        rows_per_chunk = max(1, min(bh, (1 << 30) // max(per_row, 1)))
    a = a.to(accum_dtype)
    acc = torch.zeros((pq, pq), dtype=accum_dtype, device=a.device)
    for w0 in range(0, bh, rows_per_chunk):
        h = min(rows_per_chunk, bh - w0)
        x = _window_matrix(a[w0:w0 + h + p - 1], p, q)
        acc += x @ x.conj().T
    acc /= bh * bw
    return acc
