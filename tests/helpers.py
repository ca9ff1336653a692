"""Shared test helpers (checksums identical to tests/golden/make_golden.py)."""

import numpy as np


def checksum(packed: np.ndarray) -> np.ndarray:
    k = np.arange(packed.size, dtype=np.float64)
    w = np.exp(2j * np.pi * np.modf(k * 0.6180339887498949)[0])
    s = np.sum(w * packed)
    return np.array([s.real, s.imag, np.linalg.norm(packed), packed.real.sum()])


def checksum_close(a: np.ndarray, b: np.ndarray, rtol: float) -> bool:
    """Relative agreement of two checksum vectors, scaled by the norm entry."""
    scale = max(abs(b[2]), 1e-300)
    return bool(np.all(np.abs(a - b) <= rtol * scale * 4 + 1e-300))


def c4_instances():
    """The reference's C4 sweep instances (test_acceptance.py:89-99)."""
    rng = np.random.default_rng(0xA11CE)
    out = []
    for _ in range(200):
        n = int(rng.integers(1, 25))
        m = int(rng.integers(1, 25))
        p = int(rng.integers(1, n + 1))
        q = int(rng.integers(1, m + 1))
        out.append((n, m, p, q, int(rng.integers(0, 2**32))))
    return out


def ref_random(n, m, seed):
    """InputMatrix.random of the reference (core.py:124-132)."""
    rng = np.random.default_rng(seed)
    return rng.uniform(-1.0, 1.0, (n, m)) + 1j * rng.uniform(-1.0, 1.0, (n, m))
