"""GPU parity: the CUDA path (through the C ABI) against the pinned oracle and
the reference's golden vectors.  Tolerances are those of BASELINE.json's
north_star: relative Frobenius <= 1e-12 (complex128), <= 1e-5 (complex64),
and the dense result exactly Hermitian with an exactly real diagonal."""

import numpy as np
import pytest
import torch

from helpers import c4_instances, checksum, checksum_close, ref_random
from oracle import covoracle as co
from paper_1303_2285_b200 import (
    WindowSpec,
    estimate_batch,
    estimate_batch_tensor,
    estimate_combinations,
    estimate_parallel,
    estimate_tensor,
    unique_combinations,
)
from paper_1303_2285_b200.workloads import make_input, workload

pytestmark = pytest.mark.gpu

TOL64 = 1e-12
TOL32 = 1e-5


def packed_of(dense: np.ndarray) -> np.ndarray:
    r, c = np.triu_indices(dense.shape[0])
    return dense[r, c]


def assert_hermitian(dense: np.ndarray) -> None:
    assert np.array_equal(dense, dense.conj().T)
    assert np.all(dense.diagonal().imag == 0)


def test_known_answers(cuda):
    cov, counters = estimate_combinations([[2 + 1j]], WindowSpec(1, 1))
    assert cov.numpy().tolist() == [[5 + 0j]]
    assert counters.multiplications == 1
    cov, _ = estimate_combinations(np.ones((2, 2)), WindowSpec(1, 1))
    assert cov.numpy().tolist() == [[1 + 0j]]  # 4 placements / K=4
    cov, counters = estimate_combinations(np.zeros((6, 6)), WindowSpec(2, 2))
    assert not cov.numpy().any()
    assert counters.multiplications == co.um_count(6, 6, 2, 2)


def test_cfg1(cuda, golden):
    a = make_input("cfg1")
    cov, _ = estimate_combinations(a, WindowSpec(4, 4))
    got = cov.numpy()
    assert_hermitian(got)
    assert co.rel_frobenius(packed_of(got) * 841, golden["cfg1_packed"]) <= TOL64
    assert co.rel_frobenius(got, co.covariance(a, 4, 4)) <= TOL64


@pytest.mark.parametrize("shape", [(1, 1, 1, 1), (5, 1, 2, 1), (1, 6, 1, 3), (4, 4, 4, 4), (7, 5, 1, 1),
                                   (3, 2, 3, 2), (20, 20, 8, 8), (12, 11, 4, 3), (10, 9, 3, 3)])
def test_shapes(cuda, golden, shape):
    n, m, p, q = shape
    key = f"shape_{n}_{m}_{p}_{q}"
    k = (n - p + 1) * (m - q + 1)
    for mode in ("seq", "seq-opt", "par"):
        cov, _ = estimate_combinations(golden[key + "_a"], WindowSpec(p, q), mode, threads=2)
        got = cov.numpy()
        assert_hermitian(got)
        assert co.rel_frobenius(packed_of(got) * k, golden[key + "_naive"]) <= TOL64


def test_single_window_is_outer_product(cuda):
    a = ref_random(3, 2, 5)
    cov, _ = estimate_combinations(a, WindowSpec(3, 2))
    v = a.ravel(order="F")
    np.testing.assert_allclose(cov.numpy(), np.outer(v, v.conj()), rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("spectral", [False, True])
def test_c4_sweep(cuda, golden, spectral, monkeypatch):
    """All 200 seeded instances of the reference's criterion 4 (N, M <= 24);
    spectral=True forces the frequency-domain sums wherever they apply
    (COVGPU_SPECTRAL=1: P, Q >= 2, Q <= 64, clean shapes)."""
    if spectral:
        monkeypatch.setenv("COVGPU_SPECTRAL", "1")
        monkeypatch.setenv("COVGPU_SYM", "1")  # (symmetric core sums where M >= 3Q)
    worst = 0.0
    for i, (n, m, p, q, seed) in enumerate(c4_instances()):
        a = ref_random(n, m, seed)
        k = (n - p + 1) * (m - q + 1)
        got = estimate_tensor(a, WindowSpec(p, q)).cpu().numpy()
        assert_hermitian(got)
        packed = packed_of(got) * k
        assert checksum_close(checksum(packed), golden["c4_checksums"][i], 1e-11), (i, n, m, p, q)
        err = co.rel_frobenius(packed, co.estimate_packed(a, p, q))
        worst = max(worst, err)
        assert err <= TOL64, (i, n, m, p, q, err)
    print(f"C4 worst relF {worst:.3e}")


@pytest.mark.parametrize("n,m,p,q", [(32, 32, 13, 13), (64, 64, 16, 16), (40, 70, 7, 19), (70, 40, 19, 7),
                                     (33, 65, 1, 9), (65, 33, 9, 1), (100, 37, 17, 18), (18, 18, 10, 10),
                                     (34, 34, 18, 18), (31, 97, 16, 3)])
def test_medium_shapes_vs_oracle(cuda, n, m, p, q):
    a = ref_random(n, m, n * 1000 + m * 10 + p + q)
    got = estimate_tensor(a, WindowSpec(p, q)).cpu().numpy()
    assert_hermitian(got)
    assert co.rel_frobenius(got, co.covariance(a, p, q)) <= TOL64


def test_cfg2_c128(cuda, golden):
    w = workload("cfg2")
    a = make_input(w)
    got = estimate_tensor(a, WindowSpec(w.p, w.q)).cpu().numpy()
    assert_hermitian(got)
    packed = packed_of(got) * w.k
    assert co.rel_frobenius(packed[golden["cfg2_idx"]], golden["cfg2_vals"]) <= TOL64
    assert checksum_close(checksum(packed), golden["cfg2_checksum"], 1e-11)
    assert co.rel_frobenius(got, co.covariance(a, w.p, w.q)) <= TOL64


def test_cfg2_c64(cuda, golden):
    w = workload("cfg2-c64")
    a = make_input(w)
    assert a.dtype == np.complex64
    got_t = estimate_tensor(a, WindowSpec(w.p, w.q))
    assert got_t.dtype == torch.complex64
    got = got_t.cpu().numpy()
    assert_hermitian(got)
    ref = co.covariance(a.astype(np.complex128), w.p, w.q)
    err = co.rel_frobenius(got.astype(np.complex128), ref)
    print(f"cfg2-c64 relF {err:.3e}")
    assert err <= TOL32
    packed = packed_of(got.astype(np.complex128)) * w.k
    assert co.rel_frobenius(packed[golden["cfg2_c64_idx"]], golden["cfg2_c64_vals"]) <= TOL32


def test_cfg3(cuda, golden):
    w = workload("cfg3")
    a = make_input(w)
    got = estimate_tensor(a, WindowSpec(w.p, w.q)).cpu().numpy()
    assert_hermitian(got)
    packed = packed_of(got) * w.k
    assert co.rel_frobenius(packed[golden["cfg3_idx"]], golden["cfg3_vals"]) <= TOL64
    assert checksum_close(checksum(packed), golden["cfg3_checksum"], 1e-11)


def test_cfg4_batch(cuda, golden):
    w = workload("cfg4")
    stack = make_input(w)
    got = estimate_batch_tensor(stack, WindowSpec(w.p, w.q))
    assert got.shape == (w.batch, w.pq, w.pq) and got.dtype == torch.complex64
    host = got.cpu().numpy()
    for i in range(16):
        assert_hermitian(host[i])
        packed = packed_of(host[i].astype(np.complex128)) * w.k
        assert checksum_close(checksum(packed), golden["cfg4_checksums"][i], 1e-5), i
    for i in (0, 7, 511, 1023):
        ref = co.covariance(stack[i].astype(np.complex128), w.p, w.q)
        assert co.rel_frobenius(host[i].astype(np.complex128), ref) <= TOL32
    # batch equals individual runs, bitwise (test_engine.py:150-158)
    single = estimate_tensor(stack[511], WindowSpec(w.p, w.q)).cpu().numpy()
    assert np.array_equal(single, host[511])


def test_cfg5_sampled_classes(cuda, golden_cfg5):
    """Full-size cfg5: every slot of 24 stratified classes against the
    reference's own class kernel output, plus exact Hermitian structure."""
    w = workload("cfg5")
    a = make_input(w)
    got = estimate_tensor(a, WindowSpec(w.p, w.q))
    assert torch.equal(got, got.conj().T)
    assert bool((got.diagonal().imag == 0).all())
    for ci in golden_cfg5["picked"]:
        dr, dc = (int(x) for x in golden_cfg5[f"cls_{ci}"])
        s1 = max(-dr, 0)
        pv, qu = w.p - abs(dr), w.q - dc
        u = np.arange(qu)[:, None]
        v = np.arange(pv)[None, :]
        k1 = torch.as_tensor((w.p * u + s1 + v).reshape(-1), device=got.device)
        vals = got[k1, k1 + dc * w.p + dr].cpu().numpy() * w.k
        assert co.rel_frobenius(vals, golden_cfg5[f"sums_{ci}"]) <= TOL64, (ci, dr, dc)


def test_batch_list_api_bitwise(cuda):
    mats = [ref_random(10, 10, s) for s in (1, 2, 3)]
    covs = estimate_batch(mats, WindowSpec(4, 4), threads=3)
    assert len(covs) == 3
    for mat, cov in zip(mats, covs):
        single, _ = estimate_parallel(mat, WindowSpec(4, 4), threads=1)
        assert torch.equal(cov.dense(), single.dense())
    with pytest.raises(ValueError):
        estimate_batch([ref_random(8, 8, 1), ref_random(8, 7, 1)], WindowSpec(2, 2))
    with pytest.raises(ValueError):
        estimate_batch([], WindowSpec(2, 2))


def test_modes_bitwise_identical(cuda):
    a = ref_random(14, 13, 3)
    w = WindowSpec(5, 4)
    base = estimate_combinations(a, w, "seq")[0].dense()
    for mode in ("seq-opt", "par"):
        for threads in (1, 2, 7):
            assert torch.equal(estimate_combinations(a, w, mode, threads=threads)[0].dense(), base)


def test_shards_union_bitwise(cuda):
    """Class shards computed separately reassemble the full result bit for bit
    (the multi-GPU contract)."""
    from paper_1303_2285_b200.partition import partition_classes

    w = workload("cfg2")
    a = torch.as_tensor(make_input(w), device=cuda)
    win = WindowSpec(w.p, w.q)
    full = estimate_tensor(a, win)
    for g in (2, 3, 8):
        acc = torch.zeros_like(full)
        for shard in partition_classes(w.n, w.m, win, g):
            acc += estimate_tensor(a, win, class_ids=shard)
        assert torch.equal(acc, full), g


def test_validation_errors(cuda):
    with pytest.raises(ValueError):
        estimate_combinations(np.ones((3, 3)), WindowSpec(2, 2), mode="fast")
    with pytest.raises(ValueError):
        estimate_combinations(np.ones((3, 3)), WindowSpec(4, 1))
    with pytest.raises(ValueError):
        estimate_parallel(np.ones((3, 3)), WindowSpec(2, 2), threads=0)
    with pytest.raises(ValueError):
        estimate_combinations(np.ones((2, 2, 2)), WindowSpec(1, 1))
    with pytest.raises(ValueError):
        estimate_combinations(np.ones((0, 3)), WindowSpec(1, 1))
    with pytest.raises(RuntimeError):
        estimate_combinations(np.ones((3, 3)), WindowSpec(1, 1), backend="numba")


def test_counters(cuda):
    _, counters = estimate_combinations(ref_random(32, 32, 1), WindowSpec(13, 13))
    assert counters.multiplications == 207880  # test_engine.py:112-115
    assert [r[0] for r in counters.per_combination] == unique_combinations(WindowSpec(13, 13))


def test_layouts_and_compact_scatter(cuda):
    """packed / compact outputs agree bit for bit with the dense result, and
    compact shards scattered on the root rebuild it (the multi-GPU gather)."""
    from paper_1303_2285_b200 import _native
    from paper_1303_2285_b200.distributed import cuda_ops, estimate_sharded
    from paper_1303_2285_b200.engine import _run
    from paper_1303_2285_b200.partition import partition_classes

    w = workload("cfg2")
    a = torch.as_tensor(make_input(w), device=cuda)
    win = WindowSpec(w.p, w.q)
    dense = _run(a.unsqueeze(0), win)[0]
    packed = _run(a.unsqueeze(0), win, layout=_native.PACKED)[0]
    r, c = torch.triu_indices(w.pq, w.pq, device=cuda)
    assert torch.equal(packed, dense[r, c])
    ops = cuda_ops()
    shards = partition_classes(w.n, w.m, win, 4)
    comps = [ops.compute_compact(a, win, ids) for ids in shards]
    rebuilt = ops.scatter_dense(comps, shards, win, w.n, w.m, torch.complex128, cuda)
    assert torch.equal(rebuilt, dense)
    full, comp, ids = estimate_sharded(a, (w.n, w.m), win, gather=True)
    assert torch.equal(full, dense)


def test_batch_sharded_single_process(cuda):
    from paper_1303_2285_b200.distributed import estimate_batch_sharded

    stack = torch.as_tensor(make_input("cfg4")[:64], device=cuda)
    win = WindowSpec(8, 16)
    full, local, (lo, hi) = estimate_batch_sharded(stack, tuple(stack.shape), win, gather=True)
    assert (lo, hi) == (0, 64)
    assert torch.equal(full, estimate_batch_tensor(stack, win))


def test_per_class_abi_call(cuda):
    """covgpu_combination keeps the reference kernel's per-class call shape
    (combination_scratch(a, dr, dc, p, q, out), _numba_kernels.py:62-107):
    unnormalised, only that class's packed slots written."""
    import ctypes

    from paper_1303_2285_b200 import _native

    a = ref_random(20, 18, 3)
    p, q = 5, 4
    at = torch.as_tensor(a, device=cuda)
    ref = co.estimate_packed(a, p, q)
    lib = _native.lib()
    for dr, dc in [(0, 0), (2, 1), (-3, 2), (4, 3)]:
        out = torch.zeros(p * q * (p * q + 1) // 2, dtype=torch.complex128, device=cuda)
        rc = lib.covgpu_combination(ctypes.c_void_p(at.data_ptr()), 20, 18, dr, dc, p, q,
                                    ctypes.c_void_p(out.data_ptr()),
                                    ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        _native.check(rc)
        off = co.class_packed_offsets(dr, dc, p, q)
        got = out.cpu().numpy()
        assert co.rel_frobenius(got[off], ref[off]) <= 1e-13
        mask = np.ones(got.size, bool)
        mask[off] = False
        assert not got[mask].any()
    with pytest.raises(ValueError):
        _native.check(lib.covgpu_combination(ctypes.c_void_p(at.data_ptr()), 20, 18, -1, 0, p, q,
                                             ctypes.c_void_p(out.data_ptr()), None))


def test_host_buffer_path(cuda):
    """covgpu_estimate_host / Plan.execute_host: host in, host out."""
    from paper_1303_2285_b200.plan import Plan

    w = workload("cfg2-c64")
    a = torch.from_numpy(make_input(w)).reshape(1, w.n, w.m).pin_memory()
    plan = Plan(w.n, w.m, WindowSpec(w.p, w.q), dtype=torch.complex64, device=cuda)
    out = torch.empty(plan.output_elems("packed"), dtype=torch.complex64).pin_memory()
    plan.execute_host(a, out, "packed")
    dev = estimate_tensor(a[0], WindowSpec(w.p, w.q)).cpu()
    r, c = torch.triu_indices(w.pq, w.pq)
    assert torch.equal(out, dev[r, c])
    plan.close()


def test_odd_width_c64_uses_cp_async_path(cuda):
    """complex64 rows that are not 16-byte multiples fall back to the cp.async
    bulk kernel (TMA needs aligned rows); results must still match."""
    a = (ref_random(67, 45, 11)).astype(np.complex64)
    got = estimate_tensor(a, WindowSpec(9, 7)).cpu().numpy().astype(np.complex128)
    ref = co.covariance(a.astype(np.complex128), 9, 7)
    assert co.rel_frobenius(got, ref) <= TOL32


@pytest.mark.parametrize("name", ["cfg5", "cfg3"])
def test_full_size_against_gpu_gram(cuda, name):
    """Every entry of R at full BASELINE size against the independent naive
    Gram cross-check (X X^H over all K placements, cuBLAS; oracle/gpu_naive.py)."""
    from oracle.gpu_naive import covariance_gram

    w = workload(name)
    a = torch.as_tensor(make_input(w), device=cuda)
    got = estimate_tensor(a, WindowSpec(w.p, w.q))
    ref = covariance_gram(a, w.p, w.q)
    err = (torch.linalg.norm(got - ref) / torch.linalg.norm(ref)).item()
    print(f"{name} vs Gram relF {err:.3e}")
    assert err <= TOL64


def test_cfg4_all_snapshots_against_gpu_gram(cuda):
    from oracle.gpu_naive import covariance_gram

    w = workload("cfg4")
    stack = torch.as_tensor(make_input(w), device=cuda)
    got = estimate_batch_tensor(stack, WindowSpec(w.p, w.q))
    worst = 0.0
    for b in range(0, w.batch, 8):
        ref = covariance_gram(stack[b], w.p, w.q)  # up-cast to complex128
        err = (torch.linalg.norm(got[b].to(torch.complex128) - ref) / torch.linalg.norm(ref)).item()
        worst = max(worst, err)
    print(f"cfg4 worst relF vs Gram (every 8th snapshot) {worst:.3e}")
    assert worst <= TOL32


def test_exact_algebraic_properties(cuda):
    """Size-independent identities at cfg5 size: R(2A) = 4 R(A) bit for bit
    (power-of-two scaling is exact in every operation, including the Gauss
    operand sums of the tensor-core kernel); R(conj A) = conj R(A) to 1e-15
    (the 3-multiplication form rounds (a-b)(c+d) and (a+b)(c-d) differently,
    so this one is not bitwise); trace = weighted |A|^2 sum."""
    w = workload("cfg5")
    a = torch.as_tensor(make_input(w), device=cuda)
    win = WindowSpec(w.p, w.q)
    r = estimate_tensor(a, win)
    assert torch.equal(estimate_tensor(2 * a, win), 4 * r)
    rc = estimate_tensor(a.conj().resolve_conj(), win)
    assert (torch.linalg.norm(rc - r.conj()) / torch.linalg.norm(r)).item() <= 1e-15
    # trace: element (i, j) lies in cnt_r(i) * cnt_c(j) windows
    n, m, p, q = w.n, w.m, w.p, w.q
    ri = torch.arange(n, device=cuda)
    cj = torch.arange(m, device=cuda)
    cnt_r = (torch.minimum(ri, torch.tensor(n - p, device=cuda)) - torch.clamp(ri - p + 1, min=0) + 1)
    cnt_c = (torch.minimum(cj, torch.tensor(m - q, device=cuda)) - torch.clamp(cj - q + 1, min=0) + 1)
    tr = ((a.abs() ** 2) * cnt_r[:, None] * cnt_c[None, :]).sum() / w.k
    assert abs(r.diagonal().real.sum().item() - tr.item()) <= 1e-12 * tr.item()


@pytest.mark.parametrize("n,m,p,q,batch,dt", [
    (300, 20, 130, 2, 1, np.complex128),    # P > 128: warp-per-class finalize
    (70, 66, 20, 9, 3, np.complex128),      # TMA edge kernel (strip >= 16) with batch
    (70, 66, 20, 9, 5, np.complex64),       # same, FP32, even M (TMA bulk)
    (61, 45, 17, 6, 2, np.complex64),       # odd M complex64: cp.async bulk, generic edge
    (40, 37, 25, 7, 3, np.complex128),      # unclean rows (N < 2P-2): SAT path with batch
    (33, 90, 4, 50, 2, np.complex128),      # unclean columns (M < 2Q-2)
    (50, 50, 1, 1, 4, np.complex128),       # 1x1 window
])
def test_paths_batched_vs_oracle(cuda, n, m, p, q, batch, dt):
    rng = np.random.default_rng(n * 7 + m * 13 + p + q)
    stack = (rng.standard_normal((batch, n, m)) + 1j * rng.standard_normal((batch, n, m))).astype(dt)
    got = estimate_batch_tensor(stack, WindowSpec(p, q)).cpu().numpy()
    tol = TOL64 if dt == np.complex128 else TOL32
    for b in range(batch):
        assert_hermitian(got[b])
        ref = co.covariance(stack[b].astype(np.complex128), p, q)
        assert co.rel_frobenius(got[b].astype(np.complex128), ref) <= tol, b


def test_batched_layouts_and_subsets(cuda):
    """packed / compact layouts and class subsets with batch > 1 agree bit for
    bit with the dense result."""
    from paper_1303_2285_b200 import _native
    from paper_1303_2285_b200.engine import _run
    from paper_1303_2285_b200.partition import partition_classes

    rng = np.random.default_rng(5)
    stack = torch.as_tensor(rng.standard_normal((3, 64, 48)) + 1j * rng.standard_normal((3, 64, 48)),
                            device=cuda)
    win = WindowSpec(18, 7)
    dense = _run(stack, win)
    packed = _run(stack, win, layout=_native.PACKED)
    r, c = torch.triu_indices(win.stack_size, win.stack_size, device=cuda)
    assert torch.equal(packed, dense[:, r, c])
    acc = torch.zeros_like(dense)
    for ids in partition_classes(64, 48, win, 3):
        acc += _run(stack, win, class_ids=ids)
    assert torch.equal(acc, dense)


def test_capacity_guard(cuda):
    """Packed triangle beyond 2^31-1 entries is refused before any allocation
    (core.py:147-151)."""
    with pytest.raises(ValueError):
        estimate_tensor(torch.zeros((1, 65536), dtype=torch.complex128, device=cuda), WindowSpec(1, 65536))


@pytest.mark.parametrize("spectral", [False, True])
def test_random_shapes_fuzz(cuda, spectral, monkeypatch):
    """60 seeded random shapes across every kernel path (clean / SAT, TMA /
    cp.async, small / large lag groups, batch 1-3, both dtypes) against the
    C oracle port."""
    from oracle import covoracle_c

    rng = np.random.default_rng(20261020 + (7 if spectral else 0))
    if spectral:
        monkeypatch.setenv("COVGPU_SPECTRAL", "1")
        monkeypatch.setenv("COVGPU_SYM", "1")  # the symmetric core sums wherever M >= 3Q allows them
    worst = {np.complex128: 0.0, np.complex64: 0.0}
    for it in range(60):
        n = int(rng.integers(1, 160))
        m = int(rng.integers(1, 160))
        p = int(rng.integers(1, min(n, 70) + 1))
        q = int(rng.integers(1, min(m, 70) + 1))
        batch = int(rng.integers(1, 4))
        dt = np.complex128 if it % 2 == 0 else np.complex64
        stack = (rng.standard_normal((batch, n, m)) + 1j * rng.standard_normal((batch, n, m))).astype(dt)
        got = estimate_batch_tensor(stack, WindowSpec(p, q)).cpu().numpy()
        k = (n - p + 1) * (m - q + 1)
        for b in range(batch):
            assert_hermitian(got[b])
            ref = covoracle_c.estimate_packed(stack[b].astype(np.complex128), p, q) / k
            err = co.rel_frobenius(packed_of(got[b].astype(np.complex128)), ref)
            worst[dt] = max(worst[dt], err)
            assert err <= (TOL64 if dt == np.complex128 else TOL32), (it, n, m, p, q, batch, dt, err)
    print(f"fuzz worst relF: c128 {worst[np.complex128]:.2e}, c64 {worst[np.complex64]:.2e}")


def test_integration_md_option_a(cuda, golden):
    """The ctypes binding shown in INTEGRATION.md (Option A): host buffers,
    scale 1.0 -> the reference's own unnormalised packed triangle."""
    import ctypes

    from paper_1303_2285_b200 import _native

    lib = ctypes.CDLL(str(_native.lib_path()))
    lib.covgpu_estimate_host.argtypes = [
        ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32,
        ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_double, ctypes.c_void_p,
        ctypes.c_int]
    a = np.ascontiguousarray(make_input("cfg1"), dtype=np.complex128)
    out = np.zeros(16 * 17 // 2, dtype=np.complex128)
    rc = lib.covgpu_estimate_host(a.ctypes.data, 1, 32, 32, 4, 4, 0, 1, 1.0, out.ctypes.data, 0)
    assert rc == 0
    assert co.rel_frobenius(out, golden["cfg1_packed"]) <= 1e-13
    bad = lib.covgpu_estimate_host(a.ctypes.data, 1, 32, 32, 40, 4, 0, 1, 1.0, out.ctypes.data, 0)
    assert bad == -1  # COVGPU_EINVAL -> ValueError in the binding


def test_pipelined_host_path_bitwise(cuda):
    """Batched host path (sub-batches through 3 streams) equals the device
    path bit for bit, for dense and packed outputs and a ragged last chunk."""
    from paper_1303_2285_b200.plan import Plan

    rng = np.random.default_rng(9)
    for batch in (8, 37):
        stack = (rng.standard_normal((batch, 40, 36)) + 1j * rng.standard_normal((batch, 40, 36))).astype(np.complex64)
        win = WindowSpec(6, 5)
        plan = Plan(40, 36, win, batch=batch, dtype=torch.complex64, device=cuda)
        host_a = torch.from_numpy(stack).pin_memory()
        ref = estimate_batch_tensor(stack, win).cpu()
        for layout in ("dense", "packed"):
            out = torch.empty(plan.output_elems(layout), dtype=torch.complex64).pin_memory()
            plan.execute_host(host_a, out, layout)
            if layout == "dense":
                assert torch.equal(out.reshape(batch, 30, 30), ref)
            else:
                r, c = torch.triu_indices(30, 30)
                assert torch.equal(out.reshape(batch, -1), ref[:, r, c])
        plan.close()


@pytest.mark.parametrize("n,m,p,q,batch", [
    (300, 400, 20, 40, 1),   # Q=40 in a 64-lag tile, ragged last column block
    (257, 600, 33, 70, 1),   # Q > 64: two lag tiles across dc; 3 tiles across dr
    (200, 256, 16, 24, 3),   # smallest gated window, batch of 3
    (515, 515, 32, 32, 2),   # N, M not multiples of the 16-row / 32-column chunks
])
@pytest.mark.parametrize("spectral", [False, True])
def test_tensor_core_path_vs_gram_and_cuda_cores(cuda, n, m, p, q, batch, spectral, monkeypatch):
    """complex128 core sums on the FP64 tensor cores (k_bulk_dmma) or in the
    frequency domain (spectral.cuh) against the Gram cross-check and
    against the CUDA-core bulk kernel of the same shape."""
    from oracle.gpu_naive import covariance_gram
    from paper_1303_2285_b200.plan import Plan

    rng = np.random.default_rng(n * 7 + m)
    a = torch.as_tensor(rng.standard_normal((batch, n, m)) + 1j * rng.standard_normal((batch, n, m)),
                        device=cuda)
    win = WindowSpec(p, q)
    monkeypatch.setenv("COVGPU_SPECTRAL" if spectral else "COVGPU_NO_SPECTRAL", "1")
    plan = Plan(n, m, win, batch=batch, dtype=torch.complex128, device=cuda)
    monkeypatch.delenv("COVGPU_NO_SPECTRAL", raising=False)
    monkeypatch.delenv("COVGPU_SPECTRAL", raising=False)
    plan.set_timing(True)
    got = plan.alloc_output()
    plan.execute(a, got)
    got = got.reshape(batch, p * q, p * q)
    names = plan.kernel_names()
    assert ("spec_dft" in names) == spectral, names
    assert ("bulk_dmma" in names) == (not spectral), names
    plan.close()
    monkeypatch.setenv("COVGPU_NO_MMA", "1")
    plan2 = Plan(n, m, win, batch=batch, dtype=torch.complex128, device=cuda)
    plan2.set_timing(True)
    ref_cc = plan2.alloc_output()
    plan2.execute(a, ref_cc)
    ref_cc = ref_cc.reshape(batch, p * q, p * q)
    assert "bulk_dmma" not in plan2.kernel_names()
    plan2.close()
    for b in range(batch):
        assert_hermitian(got[b].cpu().numpy())
        ref = covariance_gram(a[b], p, q)
        err = (torch.linalg.norm(got[b] - ref) / torch.linalg.norm(ref)).item()
        err_cc = (torch.linalg.norm(got[b] - ref_cc[b]) / torch.linalg.norm(ref_cc[b])).item()
        assert err <= TOL64, err
        assert err_cc <= 1e-13, err_cc


@pytest.mark.parametrize("n,m,p,q,spectral", [(1024, 1024, 64, 64, True), (1500, 900, 40, 50, True),
                                              (1024, 1024, 64, 64, False),
                                              (1536, 1536, 64, 64, True),   # above the gate of the symmetric core sums
                                              (1024, 1100, 33, 50, "sym")])  # the same, forced on a smaller shape
def test_host_path_streams_a_in_bands_bitwise(cuda, n, m, p, q, spectral, monkeypatch):
    """Single-snapshot host path: A is copied in row bands (spectral engine:
    edge columns and strip rows first) while the kernels run (band counter
    written by the copy stream); R must equal the device-resident result bit
    for bit, twice in a row (the band counter carries over between executes)
    and with the finalize walk chunked under the copy-out."""
    from paper_1303_2285_b200.plan import Plan

    if not spectral:
        monkeypatch.setenv("COVGPU_NO_SPECTRAL", "1")
    if spectral == "sym":
        monkeypatch.setenv("COVGPU_SYM", "1")
    rng = np.random.default_rng(5)
    a = torch.from_numpy(rng.standard_normal((1, n, m)) + 1j * rng.standard_normal((1, n, m))).pin_memory()
    win = WindowSpec(p, q)
    plan = Plan(n, m, win, dtype=torch.complex128, device=cuda)
    assert plan.spectral == bool(spectral)
    dev = plan.alloc_output("packed")
    plan.execute(a.to(cuda), dev, "packed")
    out = torch.empty(plan.output_elems("packed"), dtype=torch.complex128).pin_memory()
    for _ in range(2):
        out.zero_()
        plan.execute_host(a, out, "packed")
        assert torch.equal(out, dev.cpu())
    plan.close()


def test_tensor_core_path_fuzz(cuda, monkeypatch):
    """24 seeded random complex128 shapes inside the tensor-core gate (P >= 16,
    Q >= 24, wide enough M): ragged chunk / column-block / lag-tile edges,
    Q in and beyond one 64-lag tile, P above and below the tensor-core edge
    kernels' ranges, batch 1-3 — against the Gram cross-check."""
    from oracle.gpu_naive import covariance_gram
    from paper_1303_2285_b200.plan import Plan

    rng = np.random.default_rng(1303)
    worst = 0.0
    for it in range(24):
        p = int(rng.integers(16, 49))
        q = int(rng.integers(24, 49)) if it % 4 else int(rng.integers(50, 72))
        n = int(rng.integers(2 * p, 2 * p + 160))
        m = int(rng.integers(4 * q + 8, 4 * q + 200))
        batch = int(rng.integers(1, 4))
        a = torch.as_tensor(rng.standard_normal((batch, n, m)) + 1j * rng.standard_normal((batch, n, m)),
                            device=cuda)
        spectral = it % 2 == 1  # odd draws: frequency-domain sums where Q <= 64
        monkeypatch.setenv("COVGPU_SPECTRAL" if spectral else "COVGPU_NO_SPECTRAL", "1")
        plan = Plan(n, m, WindowSpec(p, q), batch=batch, dtype=torch.complex128, device=cuda)
        monkeypatch.delenv("COVGPU_NO_SPECTRAL", raising=False)
        monkeypatch.delenv("COVGPU_SPECTRAL", raising=False)
        plan.set_timing(True)
        got = plan.alloc_output()
        plan.execute(a, got)
        names = plan.kernel_names()
        if spectral:
            assert "spec_corr" in names and "spec_rc" in names, (it, n, m, p, q, names)
        else:
            assert "bulk_dmma" in names, (it, n, m, p, q, names)
        plan.close()
        got = got.reshape(batch, p * q, p * q)
        for b in range(batch):
            ref = covariance_gram(a[b], p, q)
            err = (torch.linalg.norm(got[b] - ref) / torch.linalg.norm(ref)).item()
            worst = max(worst, err)
            assert err <= TOL64, (it, n, m, p, q, batch, err)
    print(f"tensor-core fuzz worst relF {worst:.2e}")


def test_row_band_sums_and_class_range_finalize(cuda):
    """Multi-GPU row-band mode on one GPU: the sums of 3 bands added together
    (what the all-reduce does) finalize to R; one band matches the plain
    execute to rounding (the CC partials are pre-reduced in a different
    order); class-range finalizes tile the compact layout bit for bit."""
    from paper_1303_2285_b200.distributed import class_ranges
    from paper_1303_2285_b200.plan import Plan

    n, m, p, q = 400, 420, 50, 56
    rng = np.random.default_rng(77)
    a = torch.as_tensor(rng.standard_normal((n, m)) + 1j * rng.standard_normal((n, m)), device=cuda)
    win = WindowSpec(p, q)
    plan = Plan(n, m, win, dtype=torch.complex128, device=cuda)
    ref = plan.alloc_output()
    plan.execute(a, ref)
    ref_c = plan.alloc_output("compact")
    plan.execute(a, ref_c, "compact")
    # one band == the plain path up to the order of the CC partial sums
    s1 = plan.execute_sums(a, plan.alloc_sums(), 0, 1)
    got = plan.finalize_sums(a, s1, plan.alloc_output(), "dense")
    assert (torch.linalg.norm(got - ref) / torch.linalg.norm(ref)).item() <= 1e-15
    full_c = plan.finalize_sums(a, s1, plan.alloc_output("compact"), "compact")
    assert (torch.linalg.norm(full_c - ref_c) / torch.linalg.norm(ref_c)).item() <= 1e-15
    # three bands summed, each on a fresh plan (as on its own GPU: a band may
    # read only the row spectra it computed itself)
    tot = plan.alloc_sums()
    for part in range(3):
        pp = Plan(n, m, win, dtype=torch.complex128, device=cuda)
        tot += pp.execute_sums(a, pp.alloc_sums(), part, 3)
        pp.close()
    got3 = plan.finalize_sums(a, tot, plan.alloc_output(), "dense")
    err = (torch.linalg.norm(got3 - ref) / torch.linalg.norm(ref)).item()
    assert err <= 1e-14, err
    # class ranges tile the compact layout
    offs = [plan.class_slot_offset(i) for i in range(plan.num_classes + 1)]
    comp = plan.alloc_output("compact", zero=True)
    for lo, hi in class_ranges(offs, 3):
        plan.finalize_sums(a, s1, comp, "compact", lo, hi)
    assert torch.equal(comp, full_c)
    plan.close()
    # outside the tensor-core edge kernels' range the mode is refused
    small = Plan(200, 240, WindowSpec(20, 30), dtype=torch.complex128, device=cuda)
    with pytest.raises(ValueError):
        small.execute_sums(a[:200, :240].contiguous(), small.alloc_sums(), 0, 2)
    small.close()


@pytest.mark.parametrize("n,m,p,q,batch,dt", [
    (30, 40, 16, 21, 1, np.complex128),     # N = 2P-2: no core rows (dr = 0 kernel all zeros)
    (70, 62, 9, 32, 2, np.complex128),      # M = 2Q-2: no core columns beyond the edges
    (65, 129, 2, 2, 1, np.complex128),      # smallest window, FFT lengths 128 / 256 (M, N + padding)
    (200, 300, 40, 64, 1, np.complex128),   # Q = 64: the dr = 0 kernel's full 4 warps
    (257, 513, 70, 33, 1, np.complex128),   # P > 64: the L2-fed correlation kernel (9 lag groups)
    (128, 128, 8, 16, 5, np.complex64),     # cfg4 shape, complex64 inputs (FP64 spectral arithmetic)
    (100, 77, 12, 20, 3, np.complex64),
    (40, 3000, 6, 9, 1, np.complex128),     # L = 4096 after shorter lengths in this process (SMEM attribute)
    (300, 400, 20, 100, 1, np.complex128),  # Q > 64: wide edge strips (99 columns), 9801 column pairs
])
def test_spectral_path_vs_oracle(cuda, n, m, p, q, batch, dt, monkeypatch):
    """The frequency-domain sums (spectral.cuh) forced on small and ragged
    shapes against the C oracle; dense R exactly Hermitian."""
    from oracle import covoracle_c
    from paper_1303_2285_b200.plan import Plan

    monkeypatch.setenv("COVGPU_SPECTRAL", "1")
    rng = np.random.default_rng(n * 31 + m * 7 + p + q)
    stack = (rng.standard_normal((batch, n, m)) + 1j * rng.standard_normal((batch, n, m))).astype(dt)
    tdt = torch.complex128 if dt == np.complex128 else torch.complex64
    plan = Plan(n, m, WindowSpec(p, q), batch=batch, dtype=tdt, device=cuda)
    assert plan.spectral and plan.supports_rowband
    out = plan.alloc_output()
    plan.execute(torch.as_tensor(stack, device=cuda), out)
    got = out.reshape(batch, p * q, p * q).cpu().numpy()
    plan.close()
    if batch > 1:  # a snapshot's sums run in the same order alone and in a batch
        single = Plan(n, m, WindowSpec(p, q), batch=1, dtype=tdt, device=cuda)
        o1 = single.alloc_output()
        single.execute(torch.as_tensor(stack[batch - 1:], device=cuda), o1)
        assert np.array_equal(o1.reshape(p * q, p * q).cpu().numpy(), got[batch - 1])
        single.close()
    k = (n - p + 1) * (m - q + 1)
    for b in range(batch):
        assert_hermitian(got[b])
        ref = covoracle_c.estimate_packed(stack[b].astype(np.complex128), p, q) / k
        err = co.rel_frobenius(packed_of(got[b].astype(np.complex128)), ref)
        assert err <= (TOL64 if dt == np.complex128 else TOL32), (b, err)


def test_streaming_host_path_matches_sync(cuda):
    """covgpu_plan_execute_host_async: a sequence of estimates (two in flight,
    buffers reused) equals the synchronous host call bitwise."""
    from paper_1303_2285_b200.plan import Plan

    n, m, p, q = 200, 180, 20, 24
    rng = np.random.default_rng(77)
    ins = [torch.from_numpy(rng.standard_normal((1, n, m)) + 1j * rng.standard_normal((1, n, m))).pin_memory()
           for _ in range(3)]
    plan = Plan(n, m, WindowSpec(p, q), dtype=torch.complex128, device=cuda)
    ref = []
    for a in ins:
        r = torch.empty(plan.output_elems("packed"), dtype=torch.complex128).pin_memory()
        plan.execute_host(a, r, "packed")
        ref.append(r.clone())
    outs = [torch.empty(plan.output_elems("packed"), dtype=torch.complex128).pin_memory() for _ in range(2)]
    got = []
    for k, a in enumerate(ins):
        plan.execute_host_async(a, outs[k % 2], "packed")
        if k % 2 == 1:
            plan.wait()
            got += [outs[0].clone(), outs[1].clone()]
    plan.wait()
    got.append(outs[0].clone())
    plan.close()
    for r, g in zip(ref, got):
        assert torch.equal(r, g)


@pytest.mark.parametrize("n,m,p,q,force_spectral", [(32, 32, 4, 4, False), (120, 100, 12, 16, True),
                                                    (130, 140, 20, 24, "sym")])  # three streams in the graph
def test_graph_replay_bitwise(cuda, n, m, p, q, force_spectral, monkeypatch):
    """Repeated executes on the same buffers are captured into a CUDA graph
    (from the second call) and replayed; every replay reads the buffer's
    current contents and equals a graph-free plan bitwise."""
    from paper_1303_2285_b200.plan import Plan

    if force_spectral:
        monkeypatch.setenv("COVGPU_SPECTRAL", "1")
    if force_spectral == "sym":
        monkeypatch.setenv("COVGPU_SYM", "1")  # symmetric core sums: the strips' chain on the third stream
    plan = Plan(n, m, WindowSpec(p, q), dtype=torch.complex128, device=cuda)
    monkeypatch.setenv("COVGPU_NO_GRAPH", "1")
    ref_plan = Plan(n, m, WindowSpec(p, q), dtype=torch.complex128, device=cuda)
    rng = np.random.default_rng(5)
    a = torch.empty((1, n, m), dtype=torch.complex128, device=cuda)
    out = plan.alloc_output()
    ref = ref_plan.alloc_output()
    for it in range(4):
        a.copy_(torch.as_tensor(rng.standard_normal((1, n, m)) + 1j * rng.standard_normal((1, n, m))))
        plan.execute(a, out)
        ref_plan.execute(a, ref)
        torch.cuda.synchronize()
        assert torch.equal(out, ref), it
    plan.close()
    ref_plan.close()


@pytest.mark.parametrize("spectral", [False, True])
@pytest.mark.parametrize("n,m,p,q", [(200, 180, 40, 36), (150, 140, 70, 9)])
def test_wide_window_layouts_vs_oracle(cuda, spectral, n, m, p, q, monkeypatch):
    """Windows with P > 32 (two / four rows per lane in k_finalize_v): packed
    and compact R (contiguous rows per lane over the row-permuted corner
    layout) and dense R (strided rows) each match the oracle, agree with each
    other to rounding (different scan order, not bitwise), and the packed
    result is reproducible bit for bit."""
    from paper_1303_2285_b200 import _native
    from paper_1303_2285_b200.engine import _run
    if spectral and q > 64:
        pytest.skip("spectral engine needs Q <= 64")
    monkeypatch.setenv("COVGPU_SPECTRAL" if spectral else "COVGPU_NO_SPECTRAL", "1")
    a_np = ref_random(n, m, seed=n + p)
    a = torch.as_tensor(a_np, device=cuda)
    win = WindowSpec(p, q)
    k = (n - p + 1) * (m - q + 1)
    dense = _run(a.unsqueeze(0), win)[0]
    packed = _run(a.unsqueeze(0), win, layout=_native.PACKED)[0]
    packed2 = _run(a.unsqueeze(0), win, layout=_native.PACKED)[0]
    compact = _run(a.unsqueeze(0), win, layout=_native.COMPACT)[0]
    assert torch.equal(packed, packed2)
    ref = co.estimate_packed(a_np, p, q)
    assert co.rel_frobenius(packed.cpu().numpy() * k, ref) <= TOL64
    assert co.rel_frobenius(packed_of(dense.cpu().numpy()) * k, ref) <= TOL64
    r, c = torch.triu_indices(win.stack_size, win.stack_size, device=cuda)
    dpk = dense[r, c]
    assert float(torch.linalg.vector_norm(packed - dpk) / torch.linalg.vector_norm(dpk)) <= 1e-14
    assert compact.numel() == packed.numel()
    assert abs(complex(compact.sum()) - complex(packed.sum())) <= 1e-12 * float(packed.abs().sum())
    assert_hermitian(dense.cpu().numpy())


@pytest.mark.parametrize("name", ["cfg2", "cfg2-c64", "cfg3", "cfg5"])
def test_full_size_every_entry_against_c_oracle(cuda, name):
    """Every entry of R at the BASELINE size against the pinned C restatement
    of the reference's class kernel (oracle/covoracle.c, itself pinned to the
    reference's golden vectors by test_oracle.py): relF <= 1e-12 (c128) /
    1e-5 (c64, oracle on the exactly up-cast input), and the worst single
    entry relative to R's largest modulus."""
    from oracle import covoracle_c

    w = workload(name)
    a = make_input(w)
    got = estimate_tensor(a, WindowSpec(w.p, w.q)).cpu().numpy()
    assert_hermitian(got)
    ref = covoracle_c.estimate_packed(a.astype(np.complex128), w.p, w.q) / w.k
    mine = packed_of(got.astype(np.complex128))
    err = co.rel_frobenius(mine, ref)
    worst = float(np.max(np.abs(mine - ref)) / np.max(np.abs(ref)))
    print(f"{name} every entry vs C oracle: relF {err:.3e}, max entry error / max |R| {worst:.3e}")
    assert err <= (TOL64 if w.dtype == "c128" else TOL32)


def test_cfg4_every_snapshot_against_c_oracle(cuda):
    """All 1024 cfg4 snapshots, every entry, against the pinned C oracle."""
    from oracle import covoracle_c

    w = workload("cfg4")
    stack = make_input(w)
    got = estimate_batch_tensor(stack, WindowSpec(w.p, w.q)).cpu().numpy()
    worst = 0.0
    for b in range(w.batch):
        assert_hermitian(got[b])
        ref = covoracle_c.estimate_packed(stack[b].astype(np.complex128), w.p, w.q) / w.k
        err = co.rel_frobenius(packed_of(got[b].astype(np.complex128)), ref)
        worst = max(worst, err)
    print(f"cfg4 worst relF over all {w.batch} snapshots vs C oracle {worst:.3e}")
    assert worst <= TOL32


@pytest.mark.parametrize("name", ["rowband-mid", "cfg5"])
def test_row_bands_bitwise_across_gpu_counts(cuda, name):
    """The multi-GPU row-band mode run as W ranks in one process (the
    all-to-all becomes list routing): W = 1, 2, 4, 8 give the same bits
    (fixed row parts, added in part order), the result matches the C oracle,
    and a rank whose A holds only rowband_regions of its parts (NaN
    elsewhere) produces the same bits — the row-band input split."""
    from oracle import covoracle_c
    from paper_1303_2285_b200.distributed import (ROWBAND_PARTS, part_ranges, rowband_regions,
                                                  simulate_rowband)
    from paper_1303_2285_b200.plan import Plan

    if name == "cfg5":
        w = workload("cfg5")
        a_np, n, m, p, q = make_input(w), w.n, w.m, w.p, w.q
    else:
        n, m, p, q = 400, 420, 50, 56
        rng = np.random.default_rng(77)
        a_np = rng.standard_normal((n, m)) + 1j * rng.standard_normal((n, m))
    a = torch.as_tensor(a_np, device=cuda)
    win = WindowSpec(p, q)
    ref = simulate_rowband([a], win)
    assert_hermitian(ref.cpu().numpy())
    k = (n - p + 1) * (m - q + 1)
    oracle = covoracle_c.estimate_packed(a_np, p, q) / k
    err = co.rel_frobenius(packed_of(ref.cpu().numpy()), oracle)
    print(f"{name} row bands vs C oracle relF {err:.3e}")
    assert err <= TOL64
    plan = Plan(n, m, win, dtype=torch.complex128, device=cuda)
    for world in (2, 4, 8):
        bufs = []
        for r in range(world):
            # rank r's own buffer: only the regions its parts read, NaN elsewhere
            b = torch.full((n, m), complex("nan+nanj"), dtype=torch.complex128, device=cuda)
            for r0, r1, c0, c1 in rowband_regions(plan, part_ranges(ROWBAND_PARTS, world)[r]):
                b[r0:r1, c0:c1] = a[r0:r1, c0:c1]
            bufs.append(b)
        got = simulate_rowband(bufs, win)
        assert torch.equal(got, ref), world
    plan.close()


@pytest.mark.parametrize("n,m,p,q,batch", [
    (128, 128, 8, 16, 9),    # the cfg4 shape
    (127, 125, 8, 16, 3),    # N, M ragged: last chunk partial, columns past M zero-padded
    (14, 30, 8, 16, 2),      # N = 2P-2, M = 2Q-2: no core rows / core columns, edges only
    (50, 128, 2, 2, 4),      # smallest window: one lag of each sign, one strip column
    (33, 17, 3, 9, 5),       # short rows (M << FFT length), odd sizes
    (128, 64, 7, 11, 2),
    (9, 128, 5, 16, 3),      # fewer rows than a chunk and a half
])
def test_snapshot_kernel_vs_oracle(cuda, n, m, p, q, batch, monkeypatch):
    """K2 (snap.cuh): the FP32 per-snapshot spectral sums against the C
    oracle on cfg4's shape and on ragged / degenerate small shapes; exactly
    Hermitian; a snapshot alone == the same snapshot in a batch, packed ==
    dense upper triangle, and the CUDA-core engine (COVGPU_NO_SNAP=1) agrees
    within the complex64 tolerance."""
    from oracle import covoracle_c
    from paper_1303_2285_b200.plan import Plan

    rng = np.random.default_rng(n * 131 + m * 17 + p * 5 + q)
    stack = (rng.standard_normal((batch, n, m)) + 1j * rng.standard_normal((batch, n, m))).astype(np.complex64)
    ad = torch.as_tensor(stack, device=cuda)
    win = WindowSpec(p, q)
    plan = Plan(n, m, win, batch=batch, dtype=torch.complex64, device=cuda)
    assert plan.path & Plan.PATH_SNAPSHOT and not plan.spectral
    out = plan.alloc_output()
    plan.execute(ad, out)
    got = out.reshape(batch, p * q, p * q).cpu().numpy()
    pk = plan.alloc_output("packed")
    plan.execute(ad, pk, "packed")
    pkn = pk.reshape(batch, -1).cpu().numpy()
    plan.close()
    single = Plan(n, m, win, batch=1, dtype=torch.complex64, device=cuda)
    o1 = single.alloc_output()
    single.execute(ad[batch - 1:].contiguous(), o1)
    assert np.array_equal(o1.reshape(p * q, p * q).cpu().numpy(), got[batch - 1])
    single.close()
    monkeypatch.setenv("COVGPU_NO_SNAP", "1")
    direct = Plan(n, m, win, batch=batch, dtype=torch.complex64, device=cuda)
    assert not direct.path & Plan.PATH_SNAPSHOT
    od = direct.alloc_output()
    direct.execute(ad, od)
    gd = od.reshape(batch, p * q, p * q).cpu().numpy()
    direct.close()
    k = (n - p + 1) * (m - q + 1)
    for b in range(batch):
        assert_hermitian(got[b])
        assert np.array_equal(packed_of(got[b]), pkn[b])
        ref = covoracle_c.estimate_packed(stack[b].astype(np.complex128), p, q) / k
        err = co.rel_frobenius(packed_of(got[b].astype(np.complex128)), ref)
        assert err <= TOL32, (b, err)
        assert co.rel_frobenius(got[b].astype(np.complex128), gd[b].astype(np.complex128)) <= TOL32


@pytest.mark.parametrize("n,m,p,q,batch,dt", [
    (96, 120, 12, 10, 1, np.complex128),
    (100, 77, 12, 20, 3, np.complex64),     # M just above 3Q, complex64 inputs, batch
    (70, 200, 9, 32, 2, np.complex128),     # wide strips (62 columns each side)
    (64, 96, 2, 2, 1, np.complex128),       # smallest window: one lag >= 0, 2-column strips
    (140, 200, 64, 64, 1, np.complex128),   # P = Q = 64 on few rows: M = 3Q + 8
    (257, 300, 33, 17, 1, np.complex128),   # odd sizes, P > 32
])
def test_symmetric_core_sums_vs_oracle(cuda, n, m, p, q, batch, dt, monkeypatch):
    """The symmetric core sums (one column mask, lags dr >= 0 only, the
    strips' correction as extra CC partials) forced on small and ragged
    shapes against the C oracle, and against the two-mask sums
    (COVGPU_NO_SYM=1) — cfg5 runs them by default."""
    from oracle import covoracle_c
    from paper_1303_2285_b200.plan import Plan

    monkeypatch.setenv("COVGPU_SPECTRAL", "1")
    monkeypatch.setenv("COVGPU_SYM", "1")
    rng = np.random.default_rng(n * 13 + m * 5 + p + q)
    stack = (rng.standard_normal((batch, n, m)) + 1j * rng.standard_normal((batch, n, m))).astype(dt)
    tdt = torch.complex128 if dt == np.complex128 else torch.complex64
    ad = torch.as_tensor(stack, device=cuda)
    plan = Plan(n, m, WindowSpec(p, q), batch=batch, dtype=tdt, device=cuda)
    assert plan.spectral
    out = plan.alloc_output()
    plan.execute(ad, out)
    got = out.reshape(batch, p * q, p * q).cpu().numpy()
    plan.set_timing(True)  # (the kernel names of a timed execute tell which sums ran)
    plan.execute(ad, out)
    assert "spec_strips" in plan.kernel_names()
    assert np.array_equal(out.reshape(batch, p * q, p * q).cpu().numpy(), got)
    plan.set_timing(False)
    pk = plan.alloc_output("packed")
    plan.execute(ad, pk, "packed")
    pkn = pk.reshape(batch, -1).cpu().numpy()
    plan.close()
    monkeypatch.delenv("COVGPU_SYM")
    monkeypatch.setenv("COVGPU_NO_SYM", "1")
    two = Plan(n, m, WindowSpec(p, q), batch=batch, dtype=tdt, device=cuda)
    o2 = two.alloc_output()
    two.set_timing(True)
    two.execute(ad, o2)
    assert "spec_strips" not in two.kernel_names() and "spec_corr" in two.kernel_names()
    g2 = o2.reshape(batch, p * q, p * q).cpu().numpy()
    two.close()
    k = (n - p + 1) * (m - q + 1)
    tol = TOL64 if dt == np.complex128 else TOL32
    for b in range(batch):
        assert_hermitian(got[b])
        assert np.array_equal(packed_of(got[b]), pkn[b])
        ref = covoracle_c.estimate_packed(stack[b].astype(np.complex128), p, q) / k
        assert co.rel_frobenius(packed_of(got[b].astype(np.complex128)), ref) <= tol, b
        assert co.rel_frobenius(got[b].astype(np.complex128), g2[b].astype(np.complex128)) <= tol


@pytest.mark.gpu
@pytest.mark.parametrize("n,m,p,q,batch,dt", [
    (140, 200, 64, 64, 1, np.complex128),   # cfg5's window: three chunks of 16 steps at dc = 0
    (150, 120, 32, 32, 2, np.complex128),   # cfg3's window, batch
    (257, 300, 33, 17, 1, np.complex128),   # P not a multiple of the 4 x 4 thread tile
    (300, 90, 70, 20, 1, np.complex128),    # P > 64: four 64 x 64 sub-blocks per unit
    (130, 140, 45, 40, 2, np.complex64),    # complex64 inputs, ragged P
])
def test_chunk_updates_tiled_equals_walk(cuda, n, m, p, q, batch, dt, monkeypatch):
    """The walk's per-chunk state updates from the register-tiled k_ck_delta
    (windows with P >= 32, the default) equal the ones the walk kernel's DELTA
    mode accumulates (COVGPU_CK_WALK=1) bitwise: same FMA sequence per entry.
    Dense, packed and a class subset; also against the C oracle."""
    from oracle import covoracle_c
    from paper_1303_2285_b200.plan import Plan

    rng = np.random.default_rng(n + 3 * m + 7 * p + q)
    stack = (rng.standard_normal((batch, n, m)) + 1j * rng.standard_normal((batch, n, m))).astype(dt)
    tdt = torch.complex128 if dt == np.complex128 else torch.complex64
    ad = torch.as_tensor(stack, device=cuda)

    def run():
        plan = Plan(n, m, WindowSpec(p, q), batch=batch, dtype=tdt, device=cuda)
        out = plan.alloc_output()
        plan.execute(ad, out)
        plan.execute(ad, out)  # (second execute: the CUDA-graph replay)
        dense = out.reshape(batch, p * q, p * q).cpu().numpy()
        pk = plan.alloc_output("packed")
        plan.execute(ad, pk, "packed")
        packed = pk.reshape(batch, -1).cpu().numpy()
        plan.close()
        return dense, packed

    d1, p1 = run()
    monkeypatch.setenv("COVGPU_CK_WALK", "1")
    d2, p2 = run()
    assert np.array_equal(d1, d2) and np.array_equal(p1, p2)
    k = (n - p + 1) * (m - q + 1)
    tol = TOL64 if dt == np.complex128 else TOL32
    for b in range(batch):
        assert_hermitian(d1[b])
        assert np.array_equal(packed_of(d1[b]), p1[b])
        ref = covoracle_c.estimate_packed(stack[b].astype(np.complex128), p, q) / k
        assert co.rel_frobenius(p1[b].astype(np.complex128), ref) <= tol, b
