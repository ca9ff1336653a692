"""Multi-process (gloo, world size 2) tests of the multi-GPU driver's
orchestration: broadcast of A, class / snapshot sharding, gather, root-side
scatter.  The per-shard compute is the CPU oracle here (test
infrastructure); on GPUs the same driver runs the CUDA library."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import covoracle as co
from paper_1303_2285_b200 import WindowSpec
from paper_1303_2285_b200.distributed import (
    BandOps,
    ShardOps,
    class_ranges,
    estimate_batch_sharded,
    part_ranges,
    simulate_rowband,
    estimate_rowband,
    estimate_sharded,
    shard_bounds,
)
from paper_1303_2285_b200.partition import partition_classes


def oracle_ops() -> ShardOps:
    def compute_compact(a, window, ids):
        arr = a.numpy()
        n, m = arr.shape
        k = (n - window.p + 1) * (m - window.q + 1)
        combos = co.unique_combinations(window.p, window.q)
        parts = [co.class_slot_sums(arr, *combos[i], window.p, window.q) for i in sorted(set(ids))]
        return torch.from_numpy(np.concatenate(parts) / k)

    def scatter_dense(compacts, id_lists, window, n, m, dtype, device):
        dim = window.stack_size
        packed = np.zeros(dim * (dim + 1) // 2, dtype=np.complex128)
        combos = co.unique_combinations(window.p, window.q)
        for comp, ids in zip(compacts, id_lists):
            pos = 0
            vals = comp.numpy()
            for i in sorted(set(ids)):
                dr, dc = combos[i]
                off = co.class_packed_offsets(dr, dc, window.p, window.q)
                packed[off] = vals[pos:pos + off.size]
                pos += off.size
        return torch.from_numpy(co.dense_from_packed(packed, dim))

    def compute_batch(a, window):
        return torch.stack([torch.from_numpy(co.covariance(x.numpy(), window.p, window.q)) for x in a])

    return ShardOps(compute_compact, scatter_dense, compute_batch)


def oracle_band_ops() -> BandOps:
    """Row-band ops on the CPU oracle.  A part's 'sums' here are the
    unnormalised slot sums over a band of window-placement rows (linear in
    the products, so adding the parts gives the full slot sums) in compact
    (UC-major) order; finalizing a class range scales its slots by 1/K — the
    same orchestration as the CUDA ops, with oracle-defined sums."""

    def offsets_for(window):
        offs = [0]
        for dr, dc in co.unique_combinations(window.p, window.q):
            offs.append(offs[-1] + (window.p - abs(dr)) * (window.q - dc))
        return offs

    def slot_offsets(a, window):
        return offsets_for(window)

    def compute_sums(a, window, part, nparts):
        arr = a.numpy()
        n = arr.shape[0]
        bh = n - window.p + 1
        w0, w1 = bh * part // nparts, bh * (part + 1) // nparts
        sub = arr[w0:w1 + window.p - 1]
        parts = []
        for dr, dc in co.unique_combinations(window.p, window.q):
            if w1 > w0:
                parts.append(co.class_slot_sums(sub, dr, dc, window.p, window.q))
            else:
                parts.append(np.zeros((window.p - abs(dr)) * (window.q - dc), dtype=np.complex128))
        return torch.from_numpy(np.concatenate(parts))

    def sums_slices(a, window, lo, hi):
        offs = offsets_for(window)
        return [(offs[lo], offs[hi])]

    def finalize_range(a, window, sums, lo, hi):
        n, m = a.shape
        k = (n - window.p + 1) * (m - window.q + 1)
        offs = offsets_for(window)
        return sums[offs[lo]:offs[hi]] / k

    def expand_dense(compact, window, n, m, dtype, device):
        nuc = len(co.unique_combinations(window.p, window.q))
        return oracle_ops().scatter_dense([compact], [list(range(nuc))], window, n, m, dtype, device)

    return BandOps(slot_offsets, compute_sums, sums_slices, finalize_range, expand_dense)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(7)
        n, m, p, q = 20, 18, 5, 4
        a = torch.from_numpy(rng.standard_normal((n, m)) + 1j * rng.standard_normal((n, m)))
        dense, comp, ids = estimate_sharded(a if rank == 0 else None, (n, m), WindowSpec(p, q),
                                            gather=True, ops=oracle_ops(), device=torch.device("cpu"))
        out = {"ids": ids, "n_comp": int(comp.numel())}
        if rank == 0:
            ref = co.covariance(a.numpy(), p, q)
            out["err"] = co.rel_frobenius(dense.numpy(), ref)
            out["herm"] = bool(np.array_equal(dense.numpy(), dense.numpy().conj().T))
        b, n2, m2 = 5, 12, 11
        stack = torch.from_numpy(rng.standard_normal((b, n2, m2)) + 1j * rng.standard_normal((b, n2, m2)))
        full, local, (lo, hi) = estimate_batch_sharded(stack if rank == 0 else None, (b, n2, m2),
                                                       WindowSpec(3, 4), dtype=torch.complex128,
                                                       gather=True, ops=oracle_ops(),
                                                       device=torch.device("cpu"))
        out["bounds"] = (lo, hi)
        if rank == 0:
            ref = np.stack([co.covariance(x, 3, 4) for x in stack.numpy()])
            out["batch_err"] = co.rel_frobenius(full.numpy(), ref)
        # row bands: per-band sums, all-reduce, class-range finalize, gather
        dense_b, comp_b, crange = estimate_rowband(a if rank == 0 else None, (n, m), WindowSpec(p, q),
                                                   gather=True, ops=oracle_band_ops(),
                                                   device=torch.device("cpu"))
        out["band_range"] = crange
        out["band_comp"] = comp_b.numpy()
        if rank == 0:
            out["band_err"] = co.rel_frobenius(dense_b.numpy(), co.covariance(a.numpy(), p, q))
            out["band_dense"] = dense_b.numpy()
        # a mismatching input on rank 0 is refused on every rank before the broadcast
        try:
            estimate_rowband(a.to(torch.complex64) if rank == 0 else None, (n, m), WindowSpec(p, q),
                             ops=oracle_band_ops(), device=torch.device("cpu"))
            out["mismatch"] = "accepted"
        except ValueError:
            out["mismatch"] = "refused"
        results[rank] = out
    finally:
        dist.destroy_process_group()


def test_two_rank_sharded_estimate():
    world = 2
    manager = mp.Manager()
    results = manager.dict()
    mp.spawn(_worker, args=(world, _free_port(), results), nprocs=world, join=True)
    r0, r1 = results[0], results[1]
    assert r0["err"] <= 1e-13 and r0["herm"]
    assert r0["batch_err"] <= 1e-13
    shards = partition_classes(20, 18, WindowSpec(5, 4), 2)
    assert r0["ids"] == shards[0] and r1["ids"] == shards[1]
    assert set(r0["ids"]).isdisjoint(r1["ids"])
    assert r0["bounds"] == (0, 3) and r1["bounds"] == (3, 5)
    # row bands: full R on the root, contiguous class ranges covering UC
    assert r0["band_err"] <= 1e-13
    nuc = len(co.unique_combinations(5, 4))
    assert r0["band_range"][0] == 0 and r0["band_range"][1] == r1["band_range"][0]
    assert r1["band_range"][1] == nuc
    # N-invariance: the same bits as the one-process run (fixed parts, fixed order)
    rng = np.random.default_rng(7)
    a = torch.from_numpy(rng.standard_normal((20, 18)) + 1j * rng.standard_normal((20, 18)))
    dense1, _, _ = estimate_rowband(a, (20, 18), WindowSpec(5, 4), gather=True, ops=oracle_band_ops(),
                                    device=torch.device("cpu"))
    assert np.array_equal(dense1.numpy(), r0["band_dense"])
    assert r0["mismatch"] == "refused" and r1["mismatch"] == "refused"


def test_shard_bounds_cover_batch():
    for batch in (1, 7, 1024):
        for world in (1, 2, 3, 8):
            spans = [shard_bounds(batch, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == batch
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1


def test_class_ranges_balance_slots():
    offs = [0]
    for dr, dc in co.unique_combinations(64, 64):
        offs.append(offs[-1] + (64 - abs(dr)) * (64 - dc))
    for world in (1, 2, 3, 8):
        rng = class_ranges(offs, world)
        assert rng[0][0] == 0 and rng[-1][1] == len(offs) - 1
        assert all(rng[i][1] == rng[i + 1][0] for i in range(world - 1))
        loads = [offs[h] - offs[l] for l, h in rng]
        assert max(loads) - min(loads) <= 2 * 64 * 64  # within one class of even


def test_simulated_ranks_match_one_rank_bitwise():
    """simulate_rowband (the W-rank computation in one process) gives the
    same bits for W = 1, 2, 4, 8 (the row parts are fixed, their sums added
    in part order), and the result is the covariance."""
    rng = np.random.default_rng(11)
    a = torch.from_numpy(rng.standard_normal((23, 19)) + 1j * rng.standard_normal((23, 19)))
    win = WindowSpec(5, 4)
    ref = simulate_rowband([a], win, ops=oracle_band_ops())
    assert co.rel_frobenius(ref.numpy(), co.covariance(a.numpy(), 5, 4)) <= 1e-13
    for world in (2, 4, 8):
        got = simulate_rowband([a] * world, win, ops=oracle_band_ops())
        assert torch.equal(got, ref), world


def test_part_ranges_cover_parts():
    for world in (1, 2, 3, 4, 8):
        spans = part_ranges(8, world)
        assert spans[0][0] == 0 and spans[-1][1] == 8
        assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
