"""Seeded synthetic inputs for the BASELINE.json configurations.

No public dataset is involved: the reference itself only uses seeded
generators (``core.py:124-132``).  The generators here follow BASELINE.json's
configs: numpy ``default_rng(seed)`` (PCG64); CN(0, s2) draws the real part
array first, then the imaginary part array, each scaled by sqrt(s2/2).  The
same host array feeds the CPU oracle and the GPU.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["Workload", "WORKLOADS", "cn", "make_input", "workload"]


def cn(rng: np.random.Generator, shape, var: float = 1.0) -> np.ndarray:
    """Circular complex Gaussian CN(0, var), re drawn before im."""
    re = rng.standard_normal(shape)
    im = rng.standard_normal(shape)
    return (re + 1j * im) * np.sqrt(var / 2.0)


@dataclass(frozen=True)
class Workload:
    name: str
    n: int
    m: int
    p: int
    q: int
    batch: int
    dtype: str  # "c128" | "c64"
    seed: int
    kind: str  # "cn" | "sinusoids"

    @property
    def k(self) -> int:
        return (self.n - self.p + 1) * (self.m - self.q + 1)

    @property
    def pq(self) -> int:
        return self.p * self.q

    @property
    def np_dtype(self):
        return np.complex128 if self.dtype == "c128" else np.complex64


WORKLOADS = {
    "cfg1": Workload("cfg1", 32, 32, 4, 4, 1, "c128", 0, "cn"),
    "cfg2": Workload("cfg2", 256, 256, 16, 16, 1, "c128", 1, "cn"),
    "cfg2-c64": Workload("cfg2-c64", 256, 256, 16, 16, 1, "c64", 1, "cn"),
    "cfg3": Workload("cfg3", 512, 512, 32, 32, 1, "c128", 2, "sinusoids"),
    "cfg4": Workload("cfg4", 128, 128, 8, 16, 1024, "c64", 3, "cn"),
    "cfg5": Workload("cfg5", 2048, 2048, 64, 64, 1, "c128", 4, "cn"),
}


def workload(name: str) -> Workload:
    try:
        return WORKLOADS[name]
    except KeyError:
        raise ValueError(f"unknown workload {name!r}; expected one of {sorted(WORKLOADS)}") from None


def make_input(w: Workload | str) -> np.ndarray:
    """Host array for a workload: (n, m) for batch 1, (batch, n, m) otherwise."""
    if isinstance(w, str):
        w = workload(w)
    rng = np.random.default_rng(w.seed)
    if w.kind == "sinusoids":
        # 4 unit-amplitude 2-D complex sinusoids + CN(0, 0.1) noise (config 3)
        phi = rng.uniform(0.0, 2.0 * np.pi, 4)
        wr = rng.uniform(0.0, np.pi, 4)
        wc = rng.uniform(0.0, np.pi, 4)
        noise = cn(rng, (w.n, w.m), 0.1)
        n_idx = np.arange(w.n)[:, None]
        m_idx = np.arange(w.m)[None, :]
        a = np.zeros((w.n, w.m), dtype=np.complex128)
        for k in range(4):
            a += np.exp(1j * (wr[k] * n_idx + wc[k] * m_idx + phi[k]))
        a += noise
    else:
        shape = (w.n, w.m) if w.batch == 1 else (w.batch, w.n, w.m)
        a = cn(rng, shape, 1.0)
    return np.ascontiguousarray(a.astype(w.np_dtype))
