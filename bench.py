#!/usr/bin/env python
"""Benchmark of the covgpu hot path (contract: ONE JSON line from rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg5]
    python bench.py --impl reference ...          # CPU reference arm

A step = one full estimate of R for the configured workload (default cfg5:
2048x2048 complex128, P=Q=64 — BASELINE.json's largest config, which fits one
GPU).  `value` is dense R entries per second with A resident in HBM; every
step is bracketed by a barrier and device syncs, timed with CUDA events on the
launch stream, and L2 is flushed (256 MiB write) between steps.  Under
torchrun the sums are split into a fixed number of row parts (spectral /
tensor-core plans: every rank runs its parts on the rows it holds, one
all-to-all hands each rank the slices its class range needs, the parts are
added in part order, each rank finalizes its range — R bitwise the same at
any GPU count) or the offset classes are sharded (strong scaling: total work
fixed); the time is the max over ranks.

Extra keys: `kernel_ms` / `kernel_roofline` (every kernel's CUDA-event time
and its own roofline: FP64 / FP32 kernels against the DFMA / FFMA / DMMA loop
probes measured on this GPU right before the run, memory-bound kernels against
MEASURED_PEAKS.json's HBM figure, each with its algorithmic flops or bytes),
`roofline` (the dominant kernel's entry; `traffic` = its DRAM bytes per launch
from the committed ncu capture), `tensor_core_path` / `cuda_core_path` (the
same workload on the other sum engines), `packed_output` (the same step
writing the packed upper triangle, the reference's own output layout, instead
of dense Hermitian R), `cpu_baseline` (the oracle's multithreaded C port of
the reference's class kernel on this host's cores over the FULL workload — a
batch: whole snapshots — no extrapolation), `cpu_baseline_stock` (the
unmodified reference package from baseline/_ref on a bounded sample), `e2e`
(same metric through the C ABI with pinned HOST buffers: H2D of A + compute +
D2H of the packed triangle, wall clock, mean of the K calls), `e2e_pipelined`
(the streaming form, two estimates in flight), `clocks` (nvidia-smi sampled
during the timed region).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
# the side runs on the other sum engines (tensor_core_path / cuda_core_path)
# select them through the library's test hooks; the measured default plan is
# created with no switch set
os.environ.setdefault("COVGPU_TEST_HOOKS", "1")

METRIC = "R entries/s and effective GFLOP/s vs FP64/FP32 roofline at 1/2/4/8 B200"
UNIT = "R entries/s"
L2_FLUSH_BYTES = 256 << 20


def products(w):
    """(UM, bulk-kernel products, edge-row products, corner products,
    core products) per snapshot.  bulk = core rows x all columns (the
    CUDA-core bulk kernel); core = core rows x core columns (the tensor-core
    kernel; the edge columns then come from the CUDA-core kernel)."""
    from paper_1303_2285_b200.combinations import um_count, unique_combinations
    from paper_1303_2285_b200.core import WindowSpec

    n, m, p, q = w.n, w.m, w.p, w.q
    bulk = edge = corner = core = 0
    for c in unique_combinations(WindowSpec(p, q)):
        ar, ac = p - abs(c.dr) - 1, q - c.dc - 1
        rows = n - 2 * p + 2 + abs(c.dr)
        bulk += rows * (m - c.dc)
        core += rows * (m - 2 * q + 2 + c.dc)
        edge += 2 * ar * (m - 2 * q + 2 + c.dc)
        corner += 4 * ar * ac
    return um_count(n, m, p, q), bulk, edge, corner, core


def cpu_reference(w, budget_s: float):
    """Time the oracle's C port of the reference's class kernel (SAT per
    class, pthread pool over classes like engine.py:158-190) on this host's
    cores.  One snapshot: the FULL workload (every class), no extrapolation.
    A batch: whole snapshots (every class) until >= 64 snapshots and
    `budget_s` are reached, scaled by the snapshot count.
    Returns (R entries/s, sample description, threads, seconds for the
    workload)."""
    from oracle import covoracle_c
    from paper_1303_2285_b200.workloads import make_input

    a = make_input(w)
    threads = covoracle_c.max_threads()
    entries = float(w.pq) ** 2 * w.batch
    if w.batch == 1:
        t0 = time.perf_counter()
        covoracle_c.estimate_packed(a.astype(np.complex128), w.p, w.q, None, threads)
        t = time.perf_counter() - t0
        return entries / t, (f"full workload ({w.name}: all offset classes, {w.pq}x{w.pq} R) in {t:.2f} s "
                             f"on {threads} threads, no extrapolation"), threads, t
    done, t0 = 0, time.perf_counter()
    while done < w.batch and (done < 64 or time.perf_counter() - t0 < budget_s):
        covoracle_c.estimate_packed(a[done].astype(np.complex128), w.p, w.q, None, threads)
        done += 1
    t = time.perf_counter() - t0
    t_full = t * w.batch / done
    sample = (f"{done} of {w.batch} snapshots of {w.name} (every offset class) in {t:.2f} s on {threads} "
              f"threads" + ("" if done == w.batch else f", scaled by snapshot count ({t_full:.2f} s for all)"))
    return entries / t_full, sample, threads, t_full


def stock_reference(w, budget_s: float):
    """The UNMODIFIED reference package (covcomb, installed into baseline/_ref
    from /root/reference/pkg) through its own code path on this host:
    cfg1-cfg3 the fastest stock call measured in SURVEY.md §6 (numba
    seq-opt / estimate_parallel on all cores), the whole workload; cfg4
    estimate_batch on all cores over a snapshot subset; cfg5 the stock numpy
    class kernel (engine._run_class, what measure_combination_times times,
    engine.py:258-288) over a stratified class sample, scaled by each class's
    product count (the full run is ~40 min single-threaded).  None when the
    package is not installed."""
    ref_root = ROOT / "baseline" / "_ref"
    if not (ref_root / "covcomb").exists():
        return None
    if str(ref_root) not in sys.path:
        sys.path.insert(0, str(ref_root))
    try:
        import covcomb
        from covcomb import combinations as cc_comb
        from covcomb import engine as cc_engine
    except Exception as exc:  # noqa: BLE001 — report, never fail the bench
        return {"unavailable": f"covcomb import failed: {exc}"}
    from paper_1303_2285_b200.workloads import make_input

    ncores = len(os.sched_getaffinity(0))
    a = make_input(w)
    win = covcomb.WindowSpec(w.p, w.q)
    entries = float(w.pq) ** 2 * w.batch

    def best(fn, reps=2):
        fn()  # warm (numba JIT / caches)
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            fn()
            ts.append(time.perf_counter() - t0)
        return min(ts)

    try:
        if w.name == "cfg1":
            t = best(lambda: covcomb.estimate_combinations(a, win, "seq-opt", backend="numba"), reps=5)
            call, cores, sample = "estimate_combinations(mode='seq-opt', backend='numba')", 1, "full workload"
        elif w.batch == 1 and w.name != "cfg5":
            a2 = a.astype(np.complex128)
            t = best(lambda: covcomb.estimate_parallel(a2, win, threads=ncores, backend="numba"),
                     reps=1 if w.name == "cfg3" else 2)
            call, cores, sample = f"estimate_parallel(threads={ncores}, backend='numba')", ncores, "full workload"
        elif w.batch > 1:
            nb = 64
            sub = [x.astype(np.complex128) for x in a[:nb]]
            t_sub = best(lambda: covcomb.estimate_batch(sub, win, threads=ncores, backend="numba"), reps=1)
            t = t_sub * w.batch / nb
            call, cores = f"estimate_batch(threads={ncores}, backend='numba')", ncores
            sample = f"{nb} of {w.batch} snapshots in {t_sub:.2f} s, scaled by snapshot count"
        else:
            from covcomb import backend as cc_backend
            from covcomb import core as cc_core

            mat = cc_core.as_input_matrix(a)
            name = cc_backend.resolve_backend("numpy")
            kern = cc_engine._load_kernels(name)
            combos = cc_comb.unique_combinations(win)
            mu = np.array([cc_comb.pair_count(c, w.n, w.m) for c in combos], dtype=np.float64)
            out = covcomb.CovarianceMatrix(win.stack_size).packed
            scratch = np.empty(cc_engine._max_scratch(combos, win), dtype=np.complex128)
            pane = np.empty(mat.n * mat.m, dtype=np.complex128)
            cc_engine._run_class(kern, name, mat.array, combos[0], win, out, scratch, pane)  # warm
            ids = np.linspace(0, len(combos) - 1, max(8, int(budget_s / 0.3))).round().astype(int)
            ids = np.unique(ids)
            t0 = time.perf_counter()
            for i in ids:
                cc_engine._run_class(kern, name, mat.array, combos[i], win, out, scratch, pane)
            t_s = time.perf_counter() - t0
            t = t_s * mu.sum() / mu[ids].sum()
            call, cores = "engine._run_class per class, backend='numpy' (the fastest stock path at cfg5)", 1
            sample = (f"{len(ids)} of {len(combos)} offset classes (stratified) in {t_s:.1f} s, scaled by "
                      f"product count to all classes ({t:.0f} s)")
    except Exception as exc:  # noqa: BLE001
        return {"unavailable": f"stock covcomb run failed: {exc}"}
    return {"value": entries / t, "unit": UNIT, "cores": cores, "kind": "reference", "call": call,
            "sample": sample, "seconds_for_workload": t}


class ClockSampler:
    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = Path("/tmp") / f"covgpu_clocks_{os.getpid()}_{index}.csv"

    def __enter__(self):
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=self.fh, stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.fh.close()

    def summary(self):
        if self.proc is None or not self.path.exists():
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, smax, power, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.path.read_text().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
                power.append(float(parts[2]))
            except ValueError:
                continue
            for name, val in zip(names, parts[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        load = [s for s in sm if s > 500] or sm
        return {
            "sm_mhz": statistics.median(load) if load else None,
            "sm_max_mhz": max(smax) if smax else None,
            "power_w_max": max(power) if power else None,
            "samples": len(sm),
            "reasons": sorted(reasons),
        }


def bench_config(w, layout: str, world: int = 1, rowband: bool = False, sums_mib: float = 0.0) -> dict:
    """The `config` object both arms print (same keys, same values)."""
    return {"workload": w.name, "n": w.n, "m": w.m, "p": w.p, "q": w.q, "batch": w.batch,
            "input": w.dtype, "output": layout, "l2": "flushed between steps (256 MiB write)",
            "parallelism": (f"row parts x{world}: 8 fixed row parts of the sums, one all-to-all of the slices of "
                            f"[CC|CCol|RC'] each rank's class range reads ({sums_mib:.1f} MiB received per rank), "
                            f"parts added in order, class-range finalize")
            if rowband else (f"class-shard x{world}" if world > 1 else "single GPU")}


def run_reference(args, rank: int) -> None:
    """Reference arm: the reference's algorithm (the oracle's C port of its
    SAT class kernel) on all host cores, the FULL workload every step (no
    extrapolation), plus one timing of the unmodified covcomb package."""
    from paper_1303_2285_b200.workloads import workload

    if rank != 0:
        return
    w = workload(args.config)
    for _ in range(args.warmup):
        cpu_reference(w, args.ref_budget)
    vals, samples, threads, ts = [], None, 1, []
    for _ in range(args.steps):
        v, samples, threads, t = cpu_reference(w, args.ref_budget)
        vals.append(v)
        ts.append(t)
    value = statistics.median(vals)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": float(w.pq) ** 2 * w.batch / value * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": f"synthetic ({w.name}: seeded CN(0,1)/sinusoid inputs of BASELINE.json)",
        "config": bench_config(w, args.layout, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": samples,
                         "path": "oracle C port of the reference class kernel (packed upper triangle)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "timed_seconds": sum(ts),
    }
    if not args.no_stock:
        line["stock_reference"] = stock_reference(w, args.ref_budget * 3)
    print(json.dumps(line), flush=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg5")
    ap.add_argument("--impl", default="covgpu", choices=["covgpu", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=8.0, help="seconds of CPU-baseline sample")
    ap.add_argument("--ref-budget", type=float, default=4.0,
                    help="seconds of snapshots per reference-arm step (batched configs; >= 64 snapshots)")
    ap.add_argument("--no-stock", action="store_true", help="skip the unmodified-covcomb timing")
    ap.add_argument("--layout", default="dense", choices=["dense", "packed", "compact"])
    ap.add_argument("--rowband", action="store_true",
                    help="use the multi-GPU row-band mode also at N=1 (testing)")
    ap.add_argument("--no-cuda-core", action="store_true",
                    help="skip the CUDA-core (non-tensor-core) comparison steps")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return

    import torch
    import torch.distributed as dist

    from paper_1303_2285_b200.core import WindowSpec
    from paper_1303_2285_b200.partition import partition_classes, shard_cost
    from paper_1303_2285_b200.plan import Plan, probe_dmma_peak, probe_fma_peak
    from paper_1303_2285_b200.workloads import make_input, workload

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=dev)
    w = workload(args.config)
    win = WindowSpec(w.p, w.q)
    tdt = torch.complex128 if w.dtype == "c128" else torch.complex64
    # N > 1: row bands (every rank on the spectral / tensor-core sums of its
    # parts, one all-to-all of the per-part sums' slices) where the plan supports them,
    # else class shards
    plan = Plan(w.n, w.m, win, batch=w.batch, dtype=tdt, device=dev)
    rowband = (world > 1 or args.rowband) and plan.supports_rowband
    ids = None
    if world > 1 and not rowband:
        plan.close()
        ids = partition_classes(w.n, w.m, win, world, fp64=(w.dtype == "c128"))[rank]
        plan = Plan(w.n, w.m, win, batch=w.batch, dtype=tdt, class_ids=ids, device=dev)
    layout = args.layout if world == 1 and not rowband else "compact"
    if rowband:
        # fixed row parts (distributed.ROWBAND_PARTS) whatever the GPU count:
        # this rank's run of parts, one all-to-all of the slices each rank's
        # finalize range needs, the parts added in part order (R bitwise the
        # same at any N); A is split by row bands: every rank holds (resident)
        # only the rows / strips its parts read
        from paper_1303_2285_b200 import distributed as dd

        nparts = dd.ROWBAND_PARTS
        p_lo, p_hi = dd.part_ranges(nparts, world)[rank]
        part_sums = [plan.alloc_sums() for _ in range(p_lo, p_hi)]
        sums = part_sums[0]
        offsets = [plan.class_slot_offset(i) for i in range(plan.num_classes + 1)]
        ranges = dd.class_ranges(offsets, world)
        c_lo, c_hi = ranges[rank]
        slices = [plan.sums_range(lo, hi) for lo, hi in ranges]
        width = [sum(e - b for b, e in sl) for sl in slices]
        recv_sizes = [(hi - lo) * width[rank] for lo, hi in dd.part_ranges(nparts, world)]
        regions = dd.rowband_regions(plan, (p_lo, p_hi), nparts)
    host_a = make_input(w) if (rank == 0 or rowband) else None
    a = torch.zeros((w.batch, w.n, w.m), dtype=tdt, device=dev)
    if rank == 0 and not rowband:
        a.copy_(torch.from_numpy(host_a).reshape(a.shape))
    if rowband:
        ha = torch.from_numpy(host_a).reshape(w.n, w.m)
        for r0, r1, c0, c1 in regions:
            a[0, r0:r1, c0:c1] = ha[r0:r1, c0:c1].to(dev)
    out = plan.alloc_output(layout)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev)

    # roofline denominators: FMA pipe / FP64 tensor cores measured on this GPU
    # (MEASURED_PEAKS.json carries only bf16 and HBM)
    peak = probe_fma_peak(local, fp64=(w.dtype == "c128"), seconds=1.5)
    peak_dmma = probe_dmma_peak(local, seconds=1.0) if w.dtype == "c128" else None

    a_real = torch.view_as_real(a)  # collectives on the real view (no complex dtypes in NCCL)

    def step():
        if rowband:
            for j, part in enumerate(range(p_lo, p_hi)):
                plan.execute_sums(a, part_sums[j], part, nparts)
            got = dd._all_to_all(dd._rowband_send(part_sums, slices), recv_sizes, part_sums[0])
            red = dd._rowband_reduce(got, width[rank], slices[rank], part_sums[0])
            plan.finalize_sums(a, red, out, "compact", c_lo, c_hi)
        else:
            if world > 1:
                dist.broadcast(a_real, src=0)
            plan.execute(a, out, layout)

    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize(dev)

    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    total_ms = 0.0
    with ClockSampler(local) as clocks:
        t_start = time.perf_counter()
        for _ in range(args.steps):
            flush.fill_(1)  # evict A/R from L2 between steps (untimed)
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize(dev)
            e0.record()
            step()
            e1.record()
            torch.cuda.synchronize(dev)
            total_ms += e0.elapsed_time(e1)
        # short timed regions end before nvidia-smi's first samples: keep the
        # same load running (untimed) until ~0.6 s have been sampled
        while time.perf_counter() - t_start < 0.6:
            step()
            torch.cuda.synchronize(dev)
    # per-kernel breakdown: separate steps with events between the launches
    # (kernels serialised on one stream for this, so intervals are per kernel)
    plan.set_timing(True)
    kern = []
    fin_ms = []
    for _ in range(max(3, min(args.steps, 10))):
        flush.fill_(1)
        torch.cuda.synchronize(dev)
        if rowband:
            kk = None
            for j, part in enumerate(range(p_lo, p_hi)):
                plan.execute_sums(a, part_sums[j], part, nparts)
                t_j = plan.kernel_times()
                kk = t_j if kk is None else [x + y for x, y in zip(kk, t_j)]
            kern.append(kk)
            got = dd._all_to_all(dd._rowband_send(part_sums, slices), recv_sizes, part_sums[0])
            red = dd._rowband_reduce(got, width[rank], slices[rank], part_sums[0])
            torch.cuda.synchronize(dev)
            e0.record()
            plan.finalize_sums(a, red, out, "compact", c_lo, c_hi)  # delta + tile walk of the range
            e1.record()
            torch.cuda.synchronize(dev)
            fin_ms.append(e0.elapsed_time(e1))
        else:
            plan.execute(a, out, layout)
            kern.append(plan.kernel_times())
    knames = plan.kernel_names()
    plan.set_timing(False)
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item()) / args.steps

    um, bulk_p, edge_p, corner_p, core_p = products(w)
    entries = float(w.pq) ** 2 * w.batch
    value = entries / (ms * 1e-3)
    flops = 8.0 * um * w.batch
    kt = np.array(kern) if kern and all(len(k) == len(kern[0]) for k in kern) else None
    kernel_ms = {}
    if kt is not None and kt.size:
        for name, col in zip(knames, kt.mean(axis=0)):
            kernel_ms[name] = float(col)
    if fin_ms:
        kernel_ms["finalize"] = float(np.mean(fin_ms))
    shard_frac = 1.0 if ids is None else shard_cost(w.n, w.m, win, ids) / um
    if rowband:
        shard_frac = 1.0 / world
    roof = None
    hbm_peak = None
    try:
        hbm_peak = float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"])
    except (OSError, ValueError, KeyError):
        hbm_peak = 7672.0  # B200_PROFILING.md fallback
    n, m, p, q, B = w.n, w.m, w.p, w.q, w.batch
    esz_in = 16 if w.dtype == "c128" else 8
    L = 1
    while L < m:
        L *= 2
    per_kernel = {}

    def fp_roof(name, flops, note, pk=None, pk_src=None):
        ms_k = kernel_ms[name]
        ach = flops / (ms_k * 1e-3) / 1e12
        pk = peak if pk is None else pk
        return {"bound": "fp64" if w.dtype == "c128" or name.startswith("spec") else "fp32",
                "achieved": ach, "peak": pk, "unit": "TFLOP/s", "frac": ach / pk,
                "algorithmic_flops_per_launch": flops, "work": note,
                "peak_source": pk_src or "FMA-loop probe (operand-reuse DFMA/FFMA pattern) measured on this "
                "GPU in this run (MEASURED_PEAKS.json has no FP64/FP32 figure)",
                "nominal_peak": 148 * (64 if w.dtype == "c128" or name.startswith("spec") else 128) * 2
                * 1.965e9 / 1e12}

    def hbm_roof(name, nbytes, note):
        ach = nbytes / (kernel_ms[name] * 1e-3) / 1e9
        return {"bound": "hbm", "achieved": ach, "peak": hbm_peak, "unit": "GB/s", "frac": ach / hbm_peak,
                "algorithmic_bytes_per_launch": nbytes, "work": note,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (driver-measured copy bandwidth)"}

    sf = shard_frac
    for name in kernel_ms:
        if kernel_ms[name] <= 0:
            continue
        if name == "spec_corr":
            # symmetric core sums (plans that also run the strips' correction):
            # only the lags dr > 0 are correlated, the others are conjugates
            symc = "spec_strips" in kernel_ms
            macs = sum((n - 2 * p + 2 + abs(dr)) for dr in range(1 if symc else -(p - 1), p) if dr != 0) * L * B * sf
            per_kernel[name] = fp_roof(name, 6.0 * macs, "6 flops (Gauss form: 3 real FMAs) x sum over row "
                                       "lags " + ("dr > 0 (G(-dr) = conj G(dr))" if symc else "dr != 0") +
                                       " of |core rows(dr)| x L frequencies (one complex MAC per row, "
                                       "frequency and lag)")
            per_kernel[name]["complex_mac_equivalent_tflops"] = 8.0 * macs / (kernel_ms[name] * 1e-3) / 1e12
        elif name == "spec_fft":
            if "spec_strips" in kernel_ms:
                nb = (n * m * esz_in + n * L * 16) * B
                per_kernel[name] = hbm_roof(name, nb, "A read once + the one row spectrum written (the kernel "
                                            "also runs the fused dr = 0 row transforms, k_spec_fft_ac: no HBM "
                                            "bytes of their own)")
            else:
                nb = (2 * n * m * esz_in + 2 * n * L * 16 + 2 * (p - 1) * (m * esz_in + L * 16)) * B
                per_kernel[name] = hbm_roof(name, nb, "A read twice + the X / Y row spectra written "
                                            "(+ the unmasked edge-row spectra)")
        elif name == "bulk_dmma":
            per_kernel[name] = fp_roof(name, 6.0 * core_p * B * sf,
                                       "6 flops (Gauss 3 real FMAs) x core products", pk=peak_dmma,
                                       pk_src="DMMA-loop probe (mma.sync m8n8k4 f64) measured on this GPU "
                                       "in this run")
            per_kernel[name]["bound"] = "fp64-tensor"
        elif name == "bulk":
            per_kernel[name] = fp_roof(name, 8.0 * bulk_p * B * sf, "8 flops x core-row products")
        elif name == "snap_spec":
            # K2 (snap.cuh): per snapshot the 15-lag correlation over L = 128
            # frequencies, the edge-column pair correlations (pairs of strip
            # columns x 2P-1 lags x core rows) and 2N + 2P-1 FFTs of length 128
            corr = sum((n - 2 * p + 2 + abs(dr)) for dr in range(-(p - 1), p)) * 128
            pairs = sum((n - 2 * p + 2 + abs(dr)) for dr in range(-(p - 1), p)) * (q - 1) * q
            ffts = (2 * n + 2 * p - 1) * 5 * 128 * 7
            per_kernel[name] = fp_roof(name, (8.0 * (corr + pairs) + ffts) * B * sf,
                                       "8 flops x (row-lag correlation MACs over 128 frequencies + edge-column "
                                       "pair MACs) + 5 L log2 L per FFT (2N + 2P-1 transforms), per snapshot")
        elif name in ("finalize", "expand"):
            nbytes = float(w.pq) ** 2 * esz_in * B * sf if layout == "dense" else None
            if nbytes:
                per_kernel[name] = hbm_roof(name, nbytes, "dense R written once (the walk's reads of "
                                            "the per-class sums are L2-resident and not counted)")
    if per_kernel:
        dom = max(per_kernel, key=lambda k: kernel_ms[k])
        roof = dict(per_kernel[dom])
        roof["kernel"] = {"spec_corr": "k_spec_corr_smem", "spec_fft": "k_spec_fft / k_spec_fft_ac",
                          "bulk_dmma": "k_bulk_dmma3", "bulk": "k_bulk_tma", "snap_spec": "k_snap_spec", "finalize": "k_fin_tile",
                          "expand": "k_expand"}.get(dom, dom)
        roof["share_of_step"] = kernel_ms[dom] / max(sum(kernel_ms.values()), 1e-12)
        roof["traffic"] = None
        prof = ROOT / "profiles" / f"ncu_{w.name}_summary.json"
        if prof.exists():
            try:
                summ = json.loads(prof.read_text())
                roof["traffic"] = summ.get(f"{dom}_dram_bytes_per_launch")
                wf = summ.get(f"{dom}_lsu_wavefronts_per_launch")
                if wf:
                    # the walk is bound by the L1 / LSU data pipe (1 wavefront per SM per
                    # cycle), not DRAM: the same launch against that roof
                    sm_hz = 148 * 1.965e9
                    ach = wf / (kernel_ms[dom] * 1e-3)
                    roof["lsu"] = {"wavefronts_per_launch": wf, "achieved_per_s": ach, "peak_per_s": sm_hz,
                                   "frac": ach / sm_hz, "source": summ.get(f"{dom}_lsu_note")}
            except (ValueError, OSError):
                pass

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64" if w.dtype == "c128" else "f32",
        "data": f"synthetic ({w.name}: seeded CN(0,1)/sinusoid inputs of BASELINE.json)",
        "config": bench_config(w, layout, world, rowband, sum(recv_sizes) * 16 / 2**20 if rowband else 0.0),
        "effective_gflops": flops / (ms * 1e-3) / 1e9,
        "effective_gflops_note": "8 x UM (the paper's unique products) / step time; the spectral path "
                                 "does fewer flops than that, so this is not a hardware rate",
        "kernel_ms": kernel_ms,
        "kernel_roofline": {k: {kk: v[kk] for kk in ("bound", "achieved", "unit", "frac")}
                            for k, v in per_kernel.items()},
        "gpu_launches": (plan.launches * ((p_hi - p_lo) if rowband else 1) + (3 if rowband else 0)) * args.steps,
        "roofline": roof,
        "clocks": clocks.summary(),
    }

    # the earlier paths beside it, same workload, a few steps, per-kernel
    # events — reported, not the headline: the FP64 tensor-core core sums
    # (COVGPU_NO_SPECTRAL) and the north_star's CUDA-core recurrence kernels
    # (COVGPU_NO_MMA: also the path of shapes outside the spectral gates)
    def side_path(env, lay=None):
        lay = lay or layout
        for k, v in env.items():
            os.environ[k] = v
        try:
            cplan = Plan(w.n, w.m, win, batch=w.batch, dtype=tdt, device=dev)
        finally:
            for k in env:
                del os.environ[k]
        cout = cplan.alloc_output(lay)
        for _ in range(2):
            cplan.execute(a, cout, lay)
        torch.cuda.synchronize(dev)
        tot, nst = 0.0, 5
        for _ in range(nst):
            flush.fill_(1)
            torch.cuda.synchronize(dev)
            e0.record()
            cplan.execute(a, cout, lay)
            e1.record()
            torch.cuda.synchronize(dev)
            tot += e0.elapsed_time(e1)
        cplan.set_timing(True)
        flush.fill_(1)
        torch.cuda.synchronize(dev)
        cplan.execute(a, cout, lay)
        ck = dict(zip(cplan.kernel_names(), cplan.kernel_times()))
        cplan.close()
        return tot / nst, ck

    if world == 1 and not rowband and layout == "dense":
        # the reference's own output format is the packed upper triangle
        # (core.py:60-72): the same estimate written packed, for comparison
        pms, pk = side_path({}, "packed")
        line["packed_output"] = {"ms_per_step": pms, "value": entries / (pms * 1e-3), "kernel_ms": pk,
                                 "note": "same step, R written as the packed upper triangle (the "
                                         "reference's output layout) instead of dense Hermitian R"}
    if world == 1 and not args.no_cuda_core and not rowband and "spec_corr" in kernel_ms:
        tms, tk = side_path({"COVGPU_NO_SPECTRAL": "1"})
        tach = 6.0 * core_p * w.batch / (tk["bulk_dmma"] * 1e-3) / 1e12 if tk.get("bulk_dmma") else None
        line["tensor_core_path"] = {
            "ms_per_step": tms, "value": entries / (tms * 1e-3), "kernel_ms": tk,
            "bulk_dmma_achieved_tflops": tach,
            "bulk_dmma_frac_of_dmma_probe": tach / peak_dmma if tach and peak_dmma else None,
            "note": "COVGPU_NO_SPECTRAL=1: core sums as Toeplitz GEMMs on the FP64 tensor cores "
                    "(k_bulk_dmma3, 6 flops per core product), edge sums on DMMA too"}
    if world == 1 and not args.no_cuda_core and not rowband and w.dtype == "c128":
        cms, ck = side_path({"COVGPU_NO_MMA": "1", "COVGPU_NO_SPECTRAL": "1"})
        cach = 8.0 * bulk_p * w.batch / (ck["bulk"] * 1e-3) / 1e12 if ck.get("bulk") else None
        line["cuda_core_path"] = {
            "ms_per_step": cms, "value": entries / (cms * 1e-3), "kernel_ms": ck,
            "bulk_achieved_tflops": cach,
            "bulk_frac_of_fma_probe": cach / peak if cach else None,
            "bulk_frac_of_nominal_fp64": cach / (148 * 64 * 2 * 1.965e9 / 1e12) if cach else None,
            "note": "COVGPU_NO_MMA=1 COVGPU_NO_SPECTRAL=1: core sums on the FP64 FMA pipe (k_bulk_tma), "
                    "8 flops per core-row product",
        }

    if world == 1 and not rowband and "snap_spec" in kernel_ms:
        cms, ck = side_path({"COVGPU_NO_SNAP": "1"})
        cach = 8.0 * bulk_p * w.batch / (ck["bulk"] * 1e-3) / 1e12 if ck.get("bulk") else None
        line["cuda_core_path"] = {
            "ms_per_step": cms, "value": entries / (cms * 1e-3), "kernel_ms": ck,
            "bulk_achieved_tflops": cach, "bulk_frac_of_fma_probe": cach / peak if cach else None,
            "note": "COVGPU_NO_SNAP=1: the direct FP32 CUDA-core sums (k_bulk_tma, 8 flops per core-row "
                    "product) instead of the per-snapshot spectral kernel"}

    # end to end through the C ABI with pinned host buffers
    if not args.no_e2e and rowband:
        # end to end for row bands: every rank copies (pinned H2D, its own
        # PCIe link) only the regions of A its parts read, runs its parts,
        # the all-to-all, the range finalize, and copies its compact range
        # of R back (D2H) — the host input is visible to every rank
        a_host = torch.from_numpy(host_a).reshape(w.n, w.m).pin_memory()
        lo_off, hi_off = offsets[c_lo], offsets[c_hi]
        r_host = torch.empty(hi_off - lo_off, dtype=tdt).pin_memory()
        h2d = sum((r1 - r0) * (c1 - c0) for r0, r1, c0, c1 in regions) * a_host.element_size()

        def e2e_step():
            for r0, r1, c0, c1 in regions:
                a[0, r0:r1, c0:c1].copy_(a_host[r0:r1, c0:c1], non_blocking=True)
            step()
            r_host.copy_(out[lo_off:hi_off], non_blocking=True)
            torch.cuda.synchronize(dev)

        e2e_step()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            e2e_step()
        te = torch.tensor([(time.perf_counter() - t0) / args.steps], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        esz = r_host.element_size()
        line["e2e"] = {"value": entries / float(te.item()), "unit": UNIT,
                       "h2d_bytes_per_step": h2d,
                       "d2h_bytes_per_step": r_host.numel() * esz,
                       "ms_per_step": float(te.item()) * 1e3,
                       "path": "row bands: pinned H2D of the rank's regions of A (band rows + strips), "
                               "execute_sums of its parts, all-to-all, finalize_sums (class range), D2H of "
                               "the rank's compact range; wall clock, max over ranks"}
    elif not args.no_e2e:
        e2e_layout = "packed" if world == 1 else "compact"
        a_host = torch.from_numpy(host_a if rank == 0 else make_input(w)).reshape(
            w.batch, w.n, w.m).pin_memory()
        r_host = torch.empty(plan.output_elems(e2e_layout), dtype=tdt).pin_memory()
        plan.execute_host(a_host, r_host, e2e_layout)  # warm
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            plan.execute_host(a_host, r_host, e2e_layout)
        te = torch.tensor([(time.perf_counter() - t0) / args.steps], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        esz = r_host.element_size()
        line["e2e"] = {"value": entries / float(te.item()), "unit": UNIT,
                       "h2d_bytes_per_step": a_host.numel() * esz,
                       "d2h_bytes_per_step": r_host.numel() * esz,
                       "ms_per_step": float(te.item()) * 1e3,
                       "path": f"covgpu_plan_execute_host, pinned host buffers, {e2e_layout} R, wall clock"}
    if not args.no_e2e and world == 1 and w.batch < 8:
        # streaming form (covgpu_plan_execute_host_async): K estimates back to
        # back, each with its own pinned H2D of A and D2H of the packed R,
        # call k+1's copy-in and compute under call k's copy-out
        a_hosts = [torch.from_numpy(host_a).reshape(w.batch, w.n, w.m).pin_memory() for _ in range(2)]
        r_hosts = [torch.empty(plan.output_elems("packed"), dtype=tdt).pin_memory() for _ in range(2)]
        for k in range(2):
            plan.execute_host_async(a_hosts[k], r_hosts[k], "packed")
        plan.wait()
        t0 = time.perf_counter()
        for k in range(args.steps):
            plan.execute_host_async(a_hosts[k % 2], r_hosts[k % 2], "packed")
        plan.wait()
        tp = (time.perf_counter() - t0) / args.steps
        esz = r_hosts[0].element_size()
        line["e2e_pipelined"] = {
            "value": entries / tp, "unit": UNIT, "ms_per_step": tp * 1e3,
            "h2d_bytes_per_step": a_hosts[0].numel() * esz, "d2h_bytes_per_step": r_hosts[0].numel() * esz,
            "path": "covgpu_plan_execute_host_async x K then covgpu_plan_wait: every step copies its A in and "
                    "its packed R out (pinned), two estimates in flight; wall clock"}
    if rank == 0 and world == 1 and not args.no_cpu:
        v, sample, threads, t_full = cpu_reference(w, args.cpu_budget)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": threads, "kind": "port",
                                "sample": sample}
        if not args.no_stock:
            line["cpu_baseline_stock"] = stock_reference(w, args.cpu_budget)
    if rank == 0:
        print(json.dumps(line), flush=True)
    plan.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
