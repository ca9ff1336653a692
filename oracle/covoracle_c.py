"""ctypes wrapper of oracle/covoracle.c — TEST INFRASTRUCTURE ONLY.

The multithreaded C restatement of the reference's SAT class kernel
(``_numpy_kernels.py:30-53``), used for full-size parity spot checks and as
the CPU baseline in bench.py.  Pinned against the numpy oracle (and through it
the reference's golden vectors) by tests/test_oracle.py.
"""

from __future__ import annotations

import ctypes
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        path = _HERE / "libcovoracle.so"
        if not path.exists():
            subprocess.run(["make", "-C", str(_HERE)], check=True, capture_output=True)
        _LIB = ctypes.CDLL(str(path))
        _LIB.cov_class_slots.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                         ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
        _LIB.cov_estimate_packed.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                             ctypes.c_int, ctypes.c_void_p, ctypes.c_int,
                                             ctypes.c_void_p, ctypes.c_int]
        _LIB.cov_max_threads.restype = ctypes.c_int
    return _LIB


def max_threads() -> int:
    return int(lib().cov_max_threads())


def class_slots(a: np.ndarray, dr: int, dc: int, p: int, q: int) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.complex128)
    n, m = a.shape
    out = np.empty((p - abs(dr)) * (q - dc), dtype=np.complex128)
    rc = lib().cov_class_slots(a.ctypes.data, n, m, p, q, dr, dc, out.ctypes.data)
    if rc:
        raise MemoryError("cov_class_slots failed")
    return out


def estimate_packed(a: np.ndarray, p: int, q: int, class_ids=None, threads: int = 0) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.complex128)
    n, m = a.shape
    pq = p * q
    out = np.zeros(pq * (pq + 1) // 2, dtype=np.complex128)
    if class_ids is None:
        ids_p, nids = None, 0
    else:
        ids = np.ascontiguousarray(class_ids, dtype=np.int32)
        ids_p, nids = ids.ctypes.data, len(ids)
    rc = lib().cov_estimate_packed(a.ctypes.data, n, m, p, q, ids_p, nids, out.ctypes.data, threads)
    if rc:
        raise MemoryError("cov_estimate_packed failed")
    return out
