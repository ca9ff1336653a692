"""Execution plans: the reusable form of one estimate (``covgpu_plan_*`` in
include/covgpu.h).  A plan fixes the shape, dtype and class shard, owns the
device workspace, and can be executed repeatedly on device or host buffers —
what the benchmark, the multi-GPU driver and long-running callers use."""

from __future__ import annotations

import ctypes

import torch

from . import _native
from .core import WindowSpec

__all__ = ["Plan", "probe_fma_peak", "probe_dmma_peak", "LAYOUTS"]

LAYOUTS = {"dense": _native.DENSE, "packed": _native.PACKED, "compact": _native.COMPACT}
_DT = {torch.complex128: _native.C128, torch.complex64: _native.C64}


class Plan:
    def __init__(self, n: int, m: int, window: WindowSpec, batch: int = 1,
                 dtype: torch.dtype = torch.complex128, class_ids=None, device=None) -> None:
        self.lib = _native.lib()
        self.n, self.m, self.window, self.batch, self.dtype = n, m, window, batch, dtype
        self.device = torch.device(device) if device is not None else torch.device(
            "cuda", torch.cuda.current_device())
        self.class_ids = None if class_ids is None else [int(x) for x in class_ids]
        self._ids, self._nids = _native.id_array(self.class_ids)
        handle = ctypes.c_void_p()
        rc = self.lib.covgpu_plan_create(ctypes.byref(handle), self.device.index, batch, n, m,
                                         window.p, window.q, _DT[dtype], self._ids, self._nids)
        _native.check(rc, "covgpu_plan_create")
        self.handle = handle
        self._inflight = []  # host buffers of enqueued execute_host_async calls (kept alive)

    @property
    def k(self) -> int:
        return (self.n - self.window.p + 1) * (self.m - self.window.q + 1)

    def output_elems(self, layout: str = "dense") -> int:
        return int(self.lib.covgpu_output_elems(self.batch, self.n, self.m, self.window.p,
                                                self.window.q, LAYOUTS[layout], self._ids, self._nids))

    def alloc_output(self, layout: str = "dense", zero: bool = False) -> torch.Tensor:
        fn = torch.zeros if zero else torch.empty
        return fn(self.output_elems(layout), dtype=self.dtype, device=self.device)

    # ---- argument checks (the C ABI takes raw pointers and trusts sizes) ----
    def _check_input(self, a: torch.Tensor, on_device: bool) -> None:
        if a.dtype != self.dtype or not a.is_contiguous() or a.numel() != self.batch * self.n * self.m:
            raise ValueError("input does not match the plan (shape, dtype, contiguity)")
        self._check_place(a, on_device, "input")

    def _check_output(self, out: torch.Tensor, layout: str, on_device: bool) -> None:
        if layout not in LAYOUTS:
            raise ValueError(f"unknown layout {layout!r}")
        want = self.output_elems(layout)
        if out.dtype != self.dtype or not out.is_contiguous() or out.numel() != want:
            raise ValueError(f"output must be a contiguous {self.dtype} tensor of {want} elements "
                             f"({layout} layout), got {out.dtype} with {out.numel()}")
        self._check_place(out, on_device, "output")

    def _check_place(self, t: torch.Tensor, on_device: bool, what: str) -> None:
        if on_device:
            if not t.is_cuda or t.device != self.device:
                raise ValueError(f"{what} must be on {self.device}, got {t.device}")
        elif t.is_cuda:
            raise ValueError(f"{what} must be a host tensor for the host-buffer path")

    def execute(self, a: torch.Tensor, out: torch.Tensor, layout: str = "dense",
                scale: float | None = None, stream: torch.cuda.Stream | None = None) -> torch.Tensor:
        self._check_input(a, True)
        self._check_output(out, layout, True)
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        rc = self.lib.covgpu_plan_execute(self.handle, ctypes.c_void_p(a.data_ptr()),
                                          ctypes.c_void_p(out.data_ptr()), LAYOUTS[layout],
                                          1.0 / self.k if scale is None else scale,
                                          ctypes.c_void_p(st.cuda_stream))
        _native.check(rc, "covgpu_plan_execute")
        return out

    def execute_host(self, a_host: torch.Tensor, out_host: torch.Tensor, layout: str = "packed",
                     scale: float | None = None) -> torch.Tensor:
        """End to end on host buffers (pin them for full PCIe bandwidth)."""
        self._check_input(a_host, False)
        self._check_output(out_host, layout, False)
        rc = self.lib.covgpu_plan_execute_host(self.handle, ctypes.c_void_p(a_host.data_ptr()),
                                               ctypes.c_void_p(out_host.data_ptr()), LAYOUTS[layout],
                                               1.0 / self.k if scale is None else scale)
        _native.check(rc, "covgpu_plan_execute_host")
        return out_host

    def execute_host_async(self, a_host: torch.Tensor, out_host: torch.Tensor, layout: str = "packed",
                           scale: float | None = None) -> None:
        """Enqueue one host-buffer estimate (up to two in flight); the buffers
        must stay untouched until wait() returns (the plan keeps them alive)."""
        self._check_input(a_host, False)
        self._check_output(out_host, layout, False)
        self._inflight.append((a_host, out_host))
        rc = self.lib.covgpu_plan_execute_host_async(self.handle, ctypes.c_void_p(a_host.data_ptr()),
                                                     ctypes.c_void_p(out_host.data_ptr()), LAYOUTS[layout],
                                                     1.0 / self.k if scale is None else scale)
        _native.check(rc, "covgpu_plan_execute_host_async")

    def wait(self) -> None:
        rc = self.lib.covgpu_plan_wait(self.handle)
        self._inflight.clear()
        _native.check(rc, "covgpu_plan_wait")

    # ---- which sum kernels run (include/covgpu.h: covgpu_plan_path) ----
    PATH_SPECTRAL, PATH_TENSOR, PATH_ROWBAND, PATH_SNAPSHOT = 1, 2, 4, 8

    @property
    def path(self) -> int:
        f = int(self.lib.covgpu_plan_path(self.handle))
        if f < 0:
            _native.check(f, "covgpu_plan_path")
        return f

    @property
    def spectral(self) -> bool:
        return bool(self.path & self.PATH_SPECTRAL)

    @property
    def supports_rowband(self) -> bool:
        return bool(self.path & self.PATH_ROWBAND)

    # ---- multi-GPU row bands (include/covgpu.h: covgpu_plan_execute_sums) ----
    def sums_elems(self) -> int:
        """complex128 values of the reduced-sums buffer [CC | CCol | RC']."""
        return int(self.lib.covgpu_plan_sums_elems(self.handle))

    def alloc_sums(self) -> torch.Tensor:
        return torch.zeros(self.sums_elems(), dtype=torch.complex128, device=self.device)

    def execute_sums(self, a: torch.Tensor, sums: torch.Tensor, part: int = 0, nparts: int = 1,
                     stream: torch.cuda.Stream | None = None) -> torch.Tensor:
        """Part `part` of `nparts` row bands of every sum, reduced into `sums`."""
        self._check_input(a, True)
        if sums.dtype != torch.complex128 or sums.numel() != self.sums_elems() or not sums.is_contiguous():
            raise ValueError("sums buffer does not match the plan")
        self._check_place(sums, True, "sums")
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        rc = self.lib.covgpu_plan_execute_sums(self.handle, ctypes.c_void_p(a.data_ptr()),
                                               ctypes.c_void_p(sums.data_ptr()), part, nparts,
                                               ctypes.c_void_p(st.cuda_stream))
        _native.check(rc, "covgpu_plan_execute_sums")
        return sums

    def finalize_sums(self, a: torch.Tensor, sums: torch.Tensor, out: torch.Tensor,
                      layout: str = "compact", class_lo: int = 0, class_hi: int | None = None,
                      scale: float | None = None, stream: torch.cuda.Stream | None = None) -> torch.Tensor:
        """R (or the compact slots of classes [class_lo, class_hi)) from reduced sums."""
        hi = self.num_classes if class_hi is None else class_hi
        self._check_input(a, True)
        if sums.dtype != torch.complex128 or sums.numel() != self.sums_elems() or not sums.is_contiguous():
            raise ValueError("sums buffer does not match the plan")
        self._check_place(sums, True, "sums")
        if not 0 <= class_lo <= hi <= self.num_classes:
            raise ValueError("class range outside the plan")
        if layout == "compact" and (class_lo, hi) != (0, self.num_classes):
            want = self.class_slot_offset(hi) - self.class_slot_offset(class_lo)
            if out.dtype != self.dtype or not out.is_contiguous() or out.numel() < self.class_slot_offset(hi):
                raise ValueError(f"compact output must hold the plan's slots up to class {hi} "
                                 f"({self.class_slot_offset(hi)} elements; the range has {want})")
            self._check_place(out, True, "output")
        else:
            self._check_output(out, layout, True)
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        rc = self.lib.covgpu_plan_finalize_sums(
            self.handle, ctypes.c_void_p(a.data_ptr()), ctypes.c_void_p(sums.data_ptr()),
            ctypes.c_void_p(out.data_ptr()), LAYOUTS[layout], 1.0 / self.k if scale is None else scale,
            class_lo, hi, ctypes.c_void_p(st.cuda_stream))
        _native.check(rc, "covgpu_plan_finalize_sums")
        return out

    @property
    def num_classes(self) -> int:
        if self.class_ids is not None:
            return len(set(self.class_ids))
        return int(self.lib.covgpu_num_classes(self.window.p, self.window.q))

    def sums_range(self, class_lo: int, class_hi: int) -> list[tuple[int, int]]:
        """The sums-buffer slices ([CC, CCol, RC'] parts) of plan classes
        [class_lo, class_hi): what a GPU finalizing that range needs."""
        out = (ctypes.c_int64 * 6)()
        _native.check(self.lib.covgpu_plan_sums_range(self.handle, class_lo, class_hi, out),
                      "covgpu_plan_sums_range")
        return [(int(out[0]), int(out[1])), (int(out[2]), int(out[3])), (int(out[4]), int(out[5]))]

    def band_rows(self, part: int, nparts: int) -> tuple[int, int]:
        """Rows of A that execute_sums(part, nparts) reads besides the strips
        (top / bottom P-1 rows) and the first / last Q-1 columns."""
        r0, r1 = ctypes.c_int32(), ctypes.c_int32()
        _native.check(self.lib.covgpu_plan_band_rows(self.handle, part, nparts, ctypes.byref(r0),
                                                     ctypes.byref(r1)), "covgpu_plan_band_rows")
        return int(r0.value), int(r1.value)

    def class_slot_offset(self, i: int) -> int:
        """Compact offset of plan class i (i == num_classes: total slots)."""
        return int(self.lib.covgpu_plan_class_slot_offset(self.handle, i))

    def set_timing(self, enable: bool = True) -> None:
        _native.check(self.lib.covgpu_plan_set_timing(self.handle, int(enable)), "set_timing")

    def kernel_times(self) -> list[float]:
        buf = (ctypes.c_float * 12)()
        n = self.lib.covgpu_plan_kernel_times(self.handle, buf, 12)
        if n < 0:
            _native.check(n, "kernel_times")
        return [float(buf[i]) for i in range(n)]

    def kernel_names(self) -> list[str]:
        """Names of the kernel_times() intervals of the last timed execute."""
        buf = ctypes.create_string_buffer(256)
        n = self.lib.covgpu_plan_kernel_names(self.handle, buf, 256)
        if n < 0:
            _native.check(n, "kernel_names")
        return buf.value.decode().split(",") if n > 0 else []

    def kernel_timing(self) -> dict:
        """{kernel name: ms} of the last timed execute."""
        return dict(zip(self.kernel_names(), self.kernel_times()))

    @property
    def launches(self) -> int:
        return int(self.lib.covgpu_plan_launches(self.handle))

    @property
    def workspace_bytes(self) -> int:
        return int(self.lib.covgpu_plan_workspace_bytes(self.handle))

    def close(self) -> None:
        if getattr(self, "handle", None):
            self.lib.covgpu_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            self.close()
        except Exception:
            pass


def probe_fma_peak(device: int = 0, fp64: bool = True, seconds: float = 1.0) -> float:
    """Measured FMA-pipe peak (TFLOP/s) — the roofline denominator."""
    lib = _native.lib()
    out = ctypes.c_double()
    rc = lib.covgpu_probe_fma_peak(device, _native.C128 if fp64 else _native.C64, seconds,
                                   ctypes.byref(out))
    _native.check(rc, "covgpu_probe_fma_peak")
    return float(out.value)


def probe_dmma_peak(device: int = 0, seconds: float = 1.0) -> float:
    """Measured FP64 tensor-core (DMMA) peak (TFLOP/s) — the roofline
    denominator of the tensor-core bulk kernel."""
    lib = _native.lib()
    out = ctypes.c_double()
    rc = lib.covgpu_probe_dmma_peak(device, seconds, ctypes.byref(out))
    _native.check(rc, "covgpu_probe_dmma_peak")
    return float(out.value)
