"""Host-side logic on CPU: the C ABI surface, class enumeration, partitioner,
counters, validation, bench bookkeeping, and the C oracle port."""

import ctypes
import sys
import re
from pathlib import Path

import numpy as np
import pytest

from helpers import c4_instances, ref_random
from oracle import covoracle as co
from paper_1303_2285_b200 import (
    OpCounters,
    WindowSpec,
    class_index,
    estimate_batch,
    estimate_combinations,
    estimate_parallel,
    is_unique_combination,
    max_writes,
    pair_count,
    um_count,
    unique_combinations,
    work_groups,
)
from paper_1303_2285_b200 import _native
from paper_1303_2285_b200.partition import partition_classes, shard_cost

ROOT = Path(__file__).resolve().parents[1]


def header_functions():
    text = (ROOT / "include" / "covgpu.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(covgpu_[a-z_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _native.lib()  # loads libcovgpu.so (no GPU needed to dlopen)
    declared = header_functions()
    assert declared, "no functions parsed from include/covgpu.h"
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(_native.EXPORTED_SYMBOLS)


def test_host_only_entry_points():
    lib = _native.lib()
    assert lib.covgpu_num_classes(13, 13) == 313
    assert lib.covgpu_num_classes(8, 8) == 113
    assert lib.covgpu_output_elems(1, 32, 32, 4, 4, _native.DENSE, None, 0) == 256
    assert lib.covgpu_output_elems(2, 32, 32, 4, 4, _native.PACKED, None, 0) == 2 * 136
    ids = (ctypes.c_int32 * 3)(0, 5, 5)  # duplicates count once
    p, q = 4, 4
    combos = unique_combinations(WindowSpec(p, q))
    want = max_writes(combos[0], WindowSpec(p, q)) + max_writes(combos[5], WindowSpec(p, q))
    assert lib.covgpu_output_elems(1, 32, 32, p, q, _native.COMPACT, ids, 3) == want
    assert lib.covgpu_output_elems(1, 32, 32, p, q, 7, None, 0) == -1
    assert lib.covgpu_version().decode().startswith("covgpu")


def test_unique_combinations_match_reference_counts():
    assert len(unique_combinations(WindowSpec(13, 13))) == 313  # test_acceptance.py:37-47
    assert len(unique_combinations(WindowSpec(8, 8))) == 113
    assert [(c.dr, c.dc) for c in unique_combinations(WindowSpec(2, 2))] == [
        (0, 0), (0, 1), (1, 0), (1, 1), (-1, 1)]
    for p, q in [(1, 1), (3, 2), (4, 7), (13, 13)]:
        w = WindowSpec(p, q)
        combos = unique_combinations(w)
        assert [(c.dr, c.dc) for c in combos] == co.unique_combinations(p, q)
        for i, c in enumerate(combos):
            assert class_index(c.dr, c.dc, w) == i
            assert is_unique_combination(c.dr, c.dc, w)
        # eta over UC tiles the packed triangle (Eq. 4.22)
        assert sum(max_writes(c, w) for c in combos) == p * q * (p * q + 1) // 2


def test_work_groups_cover_each_class_once():
    for p, q in [(1, 1), (2, 3), (4, 4), (8, 16), (17, 5), (64, 64)]:
        w = WindowSpec(p, q)
        ids = [i for _, _, g in work_groups(w) for i in g]
        assert sorted(ids) == list(range(len(unique_combinations(w))))


@pytest.mark.parametrize("shards", [1, 2, 3, 4, 8])
def test_partition_is_disjoint_complete_and_balanced(shards):
    n, m, w = 2048, 2048, WindowSpec(64, 64)
    parts = partition_classes(n, m, w, shards)
    flat = [i for s in parts for i in s]
    assert sorted(flat) == list(range(len(unique_combinations(w))))
    costs = [shard_cost(n, m, w, s) for s in parts]
    assert sum(costs) == um_count(n, m, 64, 64)
    # 64 bulk units of ~1.6% each, LPT: within ~3% of perfect at 8 shards
    assert max(costs) <= 1.04 * sum(costs) / shards
    assert parts == partition_classes(n, m, w, shards)  # deterministic


def test_partition_units_match_library_geometry():
    import ctypes

    from paper_1303_2285_b200.partition import bulk_geometry

    lib = _native.lib()
    e, nw = ctypes.c_int32(), ctypes.c_int32()
    for n, m, p, q, batch in [(32, 32, 4, 4, 1), (256, 256, 16, 16, 1), (512, 512, 32, 32, 1),
                              (128, 128, 8, 16, 1024), (2048, 2048, 64, 64, 1), (300, 700, 100, 9, 1),
                              (20, 20, 1, 1, 1), (50, 60, 3, 2, 7), (64, 64, 5, 31, 1)]:
        for fp64 in (True, False):
            rc = lib.covgpu_bulk_geometry(batch, n, m, p, q, _native.C128 if fp64 else _native.C64,
                                          ctypes.byref(e), ctypes.byref(nw))
            assert rc == 0
            assert (e.value, nw.value) == bulk_geometry(p, fp64, n, m, q, batch), (n, m, p, q, fp64)


def test_counters_closed_form():
    w = WindowSpec(13, 13)
    c = OpCounters.tally(unique_combinations(w), w, 32, 32)
    assert c.multiplications == 207880 == um_count(32, 32, 13, 13)  # test_engine.py:112-115
    assert sum(r[1] for r in c.per_combination) == c.multiplications
    assert sum(r[2] for r in c.per_combination) == c.additions
    for comb, mults, _ in c.per_combination:
        assert mults == pair_count(comb, 32, 32)
    for n, m, p, q, _ in c4_instances()[:50]:
        assert um_count(n, m, p, q) == sum(pair_count(x, n, m) for x in unique_combinations(WindowSpec(p, q)))


def test_validation_before_device():
    with pytest.raises(ValueError):
        estimate_combinations(np.ones((3, 3)), WindowSpec(2, 2), mode="fast")
    with pytest.raises(ValueError):
        estimate_parallel(np.ones((3, 3)), WindowSpec(2, 2), threads=0)
    with pytest.raises(ValueError):
        estimate_batch([], WindowSpec(2, 2))
    with pytest.raises(ValueError):
        WindowSpec(0, 3)
    with pytest.raises(RuntimeError):
        estimate_combinations(np.ones((3, 3)), WindowSpec(1, 1), backend="numba")
    with pytest.raises(ValueError):
        estimate_combinations(np.ones((3, 3)), WindowSpec(1, 1), backend="opencl")


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        estimate_combinations(np.ones((4, 4)), WindowSpec(2, 2))


def test_bench_work_decomposition_sums_to_um():
    import bench
    from paper_1303_2285_b200.workloads import WORKLOADS

    for w in WORKLOADS.values():
        um, b, e, c, core = bench.products(w)
        assert um == b + e + c
        assert 0 < core <= b  # tensor-core core products: core rows x core columns


def test_c_oracle_matches_numpy_oracle():
    from oracle import covoracle_c

    for n, m, p, q, seed in c4_instances()[:60]:
        a = ref_random(n, m, seed)
        assert co.rel_frobenius(covoracle_c.estimate_packed(a, p, q, threads=2),
                                co.estimate_packed(a, p, q)) <= 1e-13
    a = ref_random(40, 50, 9)
    full = co.estimate_packed(a, 7, 9)
    ids = [0, 3, 17, 60, 100]
    part = covoracle_c.estimate_packed(a, 7, 9, ids)
    for i in ids:
        dr, dc = co.unique_combinations(7, 9)[i]
        off = co.class_packed_offsets(dr, dc, 7, 9)
        assert co.rel_frobenius(part[off], full[off]) <= 1e-13


@pytest.mark.parametrize("name", ["cfg2", "cfg3"])
def test_measured_gpu_cost_trace_replays_in_reference_simulator(name):
    """The per-class GPU cost trace measured on a B200 (tools/cost_trace.py:
    every class alone as a one-class plan, nothing apportioned) loads through
    the reference's own schedsim.ingest_measured_costs and replays in its
    list-scheduling simulator (schedsim.py:92-137, :174-207); its rank
    correlation with the reference's cost model mu is the committed summary."""
    import csv
    import json
    import shutil

    ref = Path("/root/reference/pkg/src/covcomb")
    if not ref.exists():
        pytest.skip("reference package not present (GPU box)")
    dst = Path("/tmp/covcomb_trace_src")
    if not dst.exists():
        shutil.copytree(ref.parent, dst)
    if str(dst) not in sys.path:
        sys.path.insert(0, str(dst))
    from covcomb import WindowSpec as RefWindow
    from covcomb import schedsim

    from paper_1303_2285_b200.workloads import workload

    w = workload(name)
    path = ROOT / "profiles" / f"r02_cost_trace_{name}.csv"
    tasks = schedsim.ingest_measured_costs(path, RefWindow(w.p, w.q))
    assert len(tasks) == len(unique_combinations(WindowSpec(w.p, w.q)))
    assert all(t.cost > 0 for t in tasks)
    with open(path) as fh:
        rows = list(csv.reader(fh))[1:]
    assert [(int(r[1]), int(r[2])) for r in rows] == [(c.dr, c.dc) for c in unique_combinations(WindowSpec(w.p, w.q))]
    lpt = schedsim.simulate(tasks, 148, "longest")
    fifo = schedsim.simulate(tasks, 148, "fifo")
    assert lpt.makespan <= fifo.makespan
    summary = json.loads((ROOT / "profiles" / f"r02_cost_trace_{name}.json").read_text())
    print(f"{name}: {len(tasks)} measured classes, spearman(cost, mu) = {summary['spearman_cost_vs_mu']:.3f}, "
          f"LPT speedup on 148 units {float(lpt.speedup):.1f}")
    assert summary["spearman_cost_vs_mu"] > 0.5
