"""Pin the CPU oracle against the reference's own outputs (tests/golden/)."""

import numpy as np
import pytest

from helpers import c4_instances, checksum, checksum_close, ref_random
from oracle import covoracle as co
from paper_1303_2285_b200.workloads import make_input, workload


def test_known_answers(golden):
    assert co.estimate_packed([[2 + 1j]], 1, 1).tolist() == [5 + 0j] == golden["ka_single"].tolist()
    assert co.naive_packed(np.ones((2, 2)), 1, 1).tolist() == golden["ka_ones"].tolist() == [4 + 0j]
    assert not co.estimate_packed(np.zeros((6, 6)), 2, 2).any()


@pytest.mark.parametrize("shape", [(1, 1, 1, 1), (5, 1, 2, 1), (1, 6, 1, 3), (4, 4, 4, 4), (7, 5, 1, 1),
                                   (3, 2, 3, 2), (20, 20, 8, 8), (12, 11, 4, 3), (10, 9, 3, 3)])
def test_shapes_match_reference(golden, shape):
    n, m, p, q = shape
    key = f"shape_{n}_{m}_{p}_{q}"
    a = golden[key + "_a"]
    assert np.array_equal(a, ref_random(n, m, n + 10 * m + 100 * p + 1000 * q))
    comb = co.estimate_packed(a, p, q)
    naive = co.naive_packed(a, p, q)
    assert co.rel_frobenius(comb, golden[key + "_comb"]) <= 1e-13
    assert co.rel_frobenius(naive, golden[key + "_naive"]) <= 1e-13


def test_c4_sweep_matches_reference(golden):
    inst = c4_instances()
    assert np.array_equal(np.array(inst, dtype=np.int64), golden["c4_params"])
    for i, (n, m, p, q, seed) in enumerate(inst):
        packed = co.estimate_packed(ref_random(n, m, seed), p, q)
        assert checksum_close(checksum(packed), golden["c4_checksums"][i], 1e-12), i
        if f"c4_{i}_packed" in golden:
            assert co.rel_frobenius(packed, golden[f"c4_{i}_packed"]) <= 1e-12


def test_cfg1_full(golden):
    assert co.rel_frobenius(co.estimate_packed(make_input("cfg1"), 4, 4), golden["cfg1_packed"]) <= 1e-13


@pytest.mark.parametrize("name", ["cfg2", "cfg2-c64"])
def test_cfg2_sampled(golden, name):
    w = workload(name)
    packed = co.estimate_packed(make_input(w).astype(np.complex128), w.p, w.q)
    key = name.replace("-", "_")
    assert co.rel_frobenius(packed[golden[key + "_idx"]], golden[key + "_vals"]) <= 1e-12
    assert checksum_close(checksum(packed), golden[key + "_checksum"], 1e-12)


def test_cfg4_snapshots(golden):
    w = workload("cfg4")
    stack = make_input(w)[:16].astype(np.complex128)
    for i in range(16):
        packed = co.estimate_packed(stack[i], w.p, w.q)
        assert checksum_close(checksum(packed), golden["cfg4_checksums"][i], 1e-12), i
    assert co.rel_frobenius(co.estimate_packed(stack[7], w.p, w.q), golden["cfg4_snap7_packed"]) <= 1e-12


def test_cfg5_classes(golden_cfg5):
    w = workload("cfg5")
    a = make_input(w)
    for ci in golden_cfg5["picked"][::6]:
        dr, dc = golden_cfg5[f"cls_{ci}"]
        sums = co.class_slot_sums(a, int(dr), int(dc), w.p, w.q)
        assert co.rel_frobenius(sums, golden_cfg5[f"sums_{ci}"]) <= 1e-12


def test_dense_is_hermitian_and_normalised():
    a = make_input("cfg1")
    r = co.covariance(a, 4, 4)
    assert np.array_equal(r, r.conj().T)
    assert np.all(r.diagonal().imag == 0)
    assert np.linalg.eigvalsh(r).min() >= -1e-12 * np.trace(r).real


def test_gpu_naive_gram_definition_on_cpu():
    """The Gram cross-check (oracle/gpu_naive.py) is the Eq. 2.2 definition:
    pin it to the class-decomposition oracle on CPU tensors."""
    import torch

    from oracle.gpu_naive import covariance_gram

    for n, m, p, q, seed in c4_instances()[:40] + [(40, 33, 7, 5, 3), (20, 20, 8, 8, 81)]:
        a = ref_random(n, m, seed)
        got = covariance_gram(torch.from_numpy(a), p, q, rows_per_chunk=3).numpy()
        assert co.rel_frobenius(got, co.covariance(a, p, q)) <= 1e-13
