"""ctypes binding of the C ABI in ``include/covgpu.h`` (libcovgpu.so).

There is no CPU fallback: if the shared library is missing or cannot be
loaded, every entry point raises ``RuntimeError`` (the reference raises
RuntimeError when its requested compiled backend is unavailable,
``backend.py:52-53``).
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

__all__ = [
    "lib",
    "lib_path",
    "check",
    "C128",
    "C64",
    "DENSE",
    "PACKED",
    "COMPACT",
    "EXPORTED_SYMBOLS",
]

C128, C64 = 0, 1
DENSE, PACKED, COMPACT = 0, 1, 2
_EINVAL, _ECUDA, _ENOMEM, _ECAPACITY = -1, -2, -3, -4

_HERE = Path(__file__).resolve().parent
LIB_NAME = "libcovgpu.so"

# every symbol include/covgpu.h declares, with (restype, argtypes)
_i64, _i32, _vp, _dbl = ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p, ctypes.c_double
_p32 = ctypes.POINTER(ctypes.c_int32)
_SIGS = {
    "covgpu_init": (ctypes.c_int, [ctypes.c_int]),
    "covgpu_last_error": (ctypes.c_char_p, []),
    "covgpu_version": (ctypes.c_char_p, []),
    "covgpu_num_classes": (_i64, [_i32, _i32]),
    "covgpu_output_elems": (_i64, [_i64, _i64, _i64, _i32, _i32, _i32, _p32, _i32]),
    "covgpu_plan_create": (
        ctypes.c_int,
        [ctypes.POINTER(_vp), ctypes.c_int, _i64, _i64, _i64, _i32, _i32, _i32, _p32, _i32],
    ),
    "covgpu_plan_execute": (ctypes.c_int, [_vp, _vp, _vp, _i32, _dbl, _vp]),
    "covgpu_plan_workspace_bytes": (_i64, [_vp]),
    "covgpu_plan_num_groups": (_i32, [_vp]),
    "covgpu_plan_launches": (_i32, [_vp]),
    "covgpu_plan_path": (_i32, [_vp]),
    "covgpu_plan_set_timing": (ctypes.c_int, [_vp, _i32]),
    "covgpu_plan_kernel_times": (_i32, [_vp, ctypes.POINTER(ctypes.c_float), _i32]),
    "covgpu_plan_kernel_names": (_i32, [_vp, ctypes.c_char_p, _i32]),
    "covgpu_plan_sums_elems": (_i64, [_vp]),
    "covgpu_plan_execute_sums": (ctypes.c_int, [_vp, _vp, _vp, _i32, _i32, _vp]),
    "covgpu_plan_finalize_sums": (ctypes.c_int, [_vp, _vp, _vp, _vp, _i32, _dbl, _i32, _i32, _vp]),
    "covgpu_plan_class_slot_offset": (_i64, [_vp, _i32]),
    "covgpu_plan_sums_range": (ctypes.c_int, [_vp, _i32, _i32, ctypes.POINTER(_i64)]),
    "covgpu_plan_band_rows": (ctypes.c_int, [_vp, _i32, _i32, _p32, _p32]),
    "covgpu_plan_destroy": (ctypes.c_int, [_vp]),
    "covgpu_estimate": (
        ctypes.c_int,
        [_vp, _i64, _i64, _i64, _i32, _i32, _i32, _i32, _p32, _i32, _dbl, _vp, _vp],
    ),
    "covgpu_estimate_host": (
        ctypes.c_int,
        [_vp, _i64, _i64, _i64, _i32, _i32, _i32, _i32, _dbl, _vp, ctypes.c_int],
    ),
    "covgpu_plan_execute_host": (ctypes.c_int, [_vp, _vp, _vp, _i32, _dbl]),
    "covgpu_plan_execute_host_async": (ctypes.c_int, [_vp, _vp, _vp, _i32, _dbl]),
    "covgpu_plan_wait": (ctypes.c_int, [_vp]),
    "covgpu_probe_fma_peak": (ctypes.c_int, [ctypes.c_int, _i32, _dbl, ctypes.POINTER(_dbl)]),
    "covgpu_probe_dmma_peak": (ctypes.c_int, [ctypes.c_int, _dbl, ctypes.POINTER(_dbl)]),
    "covgpu_bulk_geometry": (ctypes.c_int, [_i64, _i64, _i64, _i32, _i32, _i32, _p32, _p32]),
    "covgpu_scatter_compact": (
        ctypes.c_int, [_vp, _i64, _i64, _i64, _i32, _i32, _i32, _p32, _i32, _vp, _vp]),
    "covgpu_combination": (ctypes.c_int, [_vp, _i64, _i64, _i32, _i32, _i32, _i32, _vp, _vp]),
}
EXPORTED_SYMBOLS = tuple(_SIGS)

_lib = None
_load_error: str | None = None


def lib_path() -> Path:
    return Path(os.environ.get("COVGPU_LIB", _HERE / LIB_NAME))


def lib() -> ctypes.CDLL:
    """The loaded libcovgpu.so; raises RuntimeError (loudly) if unavailable."""
    global _lib, _load_error
    if _lib is not None:
        return _lib
    path = lib_path()
    if not path.exists():
        raise RuntimeError(
            f"covgpu native library not found at {path}; build it with "
            f"`python -c 'import __graft_entry__ as g; g.build()'` (there is no CPU fallback)"
        )
    try:
        handle = ctypes.CDLL(str(path))
    except OSError as exc:  # pragma: no cover - depends on the host
        _load_error = str(exc)
        raise RuntimeError(f"cannot load {path}: {exc}") from exc
    for name, (res, args) in _SIGS.items():
        fn = getattr(handle, name)
        fn.restype = res
        fn.argtypes = args
    _lib = handle
    return _lib


def last_error() -> str:
    msg = lib().covgpu_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str = "covgpu") -> None:
    """Map an ABI return code to the reference's exception types
    (ValueError for argument/capacity errors, RuntimeError otherwise)."""
    if rc == 0:
        return
    msg = f"{what}: {last_error()}"
    if rc in (_EINVAL, _ECAPACITY):
        raise ValueError(msg)
    if rc == _ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(msg)


def id_array(ids):
    """(ctypes int32 pointer, count) for a class-id list, (None, 0) for all."""
    if ids is None:
        return None, 0
    arr = (ctypes.c_int32 * len(ids))(*[int(x) for x in ids])
    return arr, len(ids)
