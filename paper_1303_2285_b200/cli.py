"""Command-line front end on the GPU path.

Mirrors the reference CLI (``cli.py:47-262``): one flat flag set dispatched
on --cmd; CSV to --out or stdout; ValueError / OSError / RuntimeError map to
exit code 2 (``cli.py:258-262``).  Commands:

  gen       seeded random input matrix (the reference generator, core.py:124-132)
  estimate  R of a file or seeded input, written in the reference text format
            (normalised by 1/K; --raw writes the reference's unnormalised sum)
  verify    GPU class decomposition vs the independent GPU naive estimator,
            and mode / thread-count bitwise invariance; exit 1 on failure
  count     closed-form operation counts (analysis.py:85-93)
  bench     CUDA-event timings per mode (+ --trace-out: per-class GPU cost trace
            in the reference's task_id,dr,dc,cost format)
"""

from __future__ import annotations

import argparse
import csv
import sys

import numpy as np

__all__ = ["main", "BENCH_HEADER", "VERIFY_HEADER", "VERIFY_TOL", "COUNT_HEADER"]

BENCH_HEADER = ["mode", "threads", "N", "M", "P", "Q", "seconds", "speedup_vs_naive", "mults", "adds"]
VERIFY_HEADER = ["comparison", "max_rel_diff", "pass"]
COUNT_HEADER = ["N", "M", "P", "Q", "SM", "SA", "UM1", "UM2", "UM", "UMHAT", "RATIO"]
VERIFY_TOL = 1e-10
_MODES = ["naive", "seq", "seq-opt", "par"]


class _CliError(Exception):
    pass


def _positive_int(text: str) -> int:
    try:
        v = int(text)
    except ValueError:
        raise argparse.ArgumentTypeError(f"expected an integer, got {text!r}") from None
    if v < 1:
        raise argparse.ArgumentTypeError(f"expected a positive integer, got {text}")
    return v


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="covgpu", description=__doc__,
                                 formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--cmd", required=True, choices=["gen", "estimate", "verify", "count", "bench"])
    ap.add_argument("--in", dest="in_path", metavar="PATH")
    ap.add_argument("--out", metavar="PATH")
    ap.add_argument("--n", type=_positive_int)
    ap.add_argument("--m", type=_positive_int)
    ap.add_argument("--p", type=_positive_int)
    ap.add_argument("--q", type=_positive_int)
    ap.add_argument("--mode", choices=_MODES)
    ap.add_argument("--threads", type=_positive_int, default=1)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--repeats", type=_positive_int, default=5)
    ap.add_argument("--backend", choices=["cuda", "auto"])
    ap.add_argument("--raw", action="store_true", help="estimate: write the unnormalised sum")
    ap.add_argument("--complex64", action="store_true", help="run the FP32 path")
    ap.add_argument("--trace-out", dest="trace_out", metavar="PATH")
    return ap


def _require(args, *names):
    miss = [f"--{n}" for n in names if getattr(args, n) is None]
    if miss:
        raise _CliError(f"--cmd {args.cmd} requires {', '.join(miss)}")


def _window(args):
    from .core import WindowSpec

    _require(args, "p", "q")
    return WindowSpec(args.p, args.q)


def _load(args) -> np.ndarray:
    from .io import read_input_matrix

    if args.in_path is not None:
        a = read_input_matrix(args.in_path)
    else:
        _require(args, "n", "m")
        rng = np.random.default_rng(args.seed)
        a = rng.uniform(-1.0, 1.0, (args.n, args.m)) + 1j * rng.uniform(-1.0, 1.0, (args.n, args.m))
    return a.astype(np.complex64) if args.complex64 else a


def _emit(header, rows, out):
    def write(fh):
        w = csv.writer(fh)
        w.writerow(header)
        for r in rows:
            w.writerow(["pass" if c is True else "fail" if c is False else
                        repr(c) if isinstance(c, float) else str(c) for c in r])
    if out is None:
        write(sys.stdout)
    else:
        with open(out, "w", newline="", encoding="utf-8") as fh:
            write(fh)


def _run_mode(a, window, mode, args):
    from . import engine
    from .naive import estimate_naive

    if mode == "naive":
        return estimate_naive(a, window), None
    cov, counters = engine.estimate_combinations(a, window, mode, threads=args.threads,
                                                 backend=args.backend)
    return cov.dense(), counters


def _cmd_gen(args):
    from .io import write_input_matrix

    _require(args, "n", "m", "out")
    write_input_matrix(_load(args), args.out)
    return 0


def _cmd_estimate(args):
    from .io import write_covariance

    _require(args, "out")
    window = _window(args)
    a = _load(args)
    dense, _ = _run_mode(a, window, args.mode or "seq-opt", args)
    if args.raw:
        dense = dense * ((a.shape[0] - window.p + 1) * (a.shape[1] - window.q + 1))
    write_covariance(dense, args.out)
    return 0


def _max_rel(a, b) -> float:
    import torch

    scale = max(float(a.abs().max()), float(b.abs().max()))
    return 0.0 if scale == 0.0 else float((a.to(torch.complex128) - b.to(torch.complex128)).abs().max()) / scale


def _cmd_verify(args):
    import torch

    from . import engine
    from .naive import estimate_naive

    window = _window(args)
    a = _load(args)
    tol = 1e-5 if args.complex64 else VERIFY_TOL
    labeled = [("naive", estimate_naive(a, window))]
    for mode in ("seq", "seq-opt"):
        labeled.append((mode, engine.estimate_combinations(a, window, mode, backend=args.backend)[0].dense()))
    labeled.append((f"par{args.threads}", engine.estimate_parallel(a, window, args.threads,
                                                                     backend=args.backend)[0].dense()))
    rows, ok_all = [], True
    for i in range(len(labeled)):
        for j in range(i + 1, len(labeled)):
            d = _max_rel(labeled[i][1], labeled[j][1])
            exact = i > 0  # GPU modes must agree bit for bit
            ok = (d == 0.0) if exact else d <= tol
            ok_all &= ok
            rows.append([f"{labeled[i][0]}_vs_{labeled[j][0]}", d, ok])
    herm = bool(torch.equal(labeled[1][1], labeled[1][1].conj().T))
    rows.append(["hermitian", 0.0 if herm else 1.0, herm])
    ok_all &= herm
    _emit(VERIFY_HEADER, rows, args.out)
    return 0 if ok_all else 1


def _cmd_count(args):
    from fractions import Fraction

    from .combinations import um_count

    _require(args, "n", "m", "p", "q")
    n, m, p, q = args.n, args.m, args.p, args.q
    if p > n or q > m:
        raise ValueError(f"{p}x{q} window does not fit a {n}x{m} matrix")
    sm = (n - p) * (m - q) * p * p * q * q  # analysis.py:54-65 (paper's exclusive factor)
    um1 = (p * (2 * n - p + 1) // 2) * (q * (2 * m - q + 1) // 2)
    um2 = ((p - 1) * (2 * n - p) // 2) * ((q - 1) * (2 * m - q) // 2)
    assert um1 + um2 == um_count(n, m, p, q)
    ratio = Fraction(sm, 2 * um1)
    _emit(COUNT_HEADER, [[n, m, p, q, sm, sm, um1, um2, um1 + um2, 2 * um1, float(ratio)]], args.out)
    return 0


def _cmd_bench(args):
    import torch

    from . import engine

    window = _window(args)
    a = _load(args)
    n, m = a.shape
    dev_a = torch.as_tensor(a, device="cuda")
    modes = [args.mode] if args.mode else list(_MODES)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def best(fn):
        fn()
        b = float("inf")
        for _ in range(args.repeats):
            e0.record()
            fn()
            e1.record()
            e1.synchronize()
            b = min(b, e0.elapsed_time(e1) * 1e-3)
        return b

    t_naive = best(lambda: _run_mode(dev_a, window, "naive", args))
    rows = []
    k = (n - window.p + 1) * (m - window.q + 1)
    tri = window.stack_size * (window.stack_size + 1) // 2
    for mode in modes:
        threads = args.threads if mode == "par" else 1
        if mode == "naive":
            secs, mults, adds = t_naive, k * tri, k * tri
        else:
            secs = best(lambda: _run_mode(dev_a, window, mode, args))
            _, c = _run_mode(dev_a, window, mode, args)
            mults, adds = c.multiplications, c.additions
        rows.append([mode, threads, n, m, window.p, window.q, secs, t_naive / secs, mults, adds])
    _emit(BENCH_HEADER, rows, args.out)
    if args.trace_out is not None:
        engine.write_cost_trace(args.trace_out,
                                engine.measure_combination_times(dev_a, window, repeats=max(3, args.repeats)))
    return 0


_DISPATCH = {"gen": _cmd_gen, "estimate": _cmd_estimate, "verify": _cmd_verify,
             "count": _cmd_count, "bench": _cmd_bench}


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return _DISPATCH[args.cmd](args)
    except (_CliError, ValueError, OSError, RuntimeError) as exc:
        print(f"covgpu: error: {exc}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
