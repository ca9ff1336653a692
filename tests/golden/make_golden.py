"""Generate the golden fixtures by running the REAL reference (``covcomb``).

Run once in the build container (the reference cannot travel to the GPU box):

    python tests/golden/make_golden.py            # everything except cfg5 classes
    python tests/golden/make_golden.py --cfg5     # also the cfg5 per-class sample

The reference is imported from a scratch copy of ``/root/reference/pkg/src``
(numba's ``cache=True`` writes next to the sources, and the mount is
read-only).  Outputs are the reference's own UNNORMALISED packed triangles;
tests apply 1/K themselves.  Large configs are stored as checksums plus a
seeded sample of packed entries so the fixtures stay small.
"""

from __future__ import annotations

import argparse
import functools
import os
import shutil
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parents[1]
sys.path.insert(0, str(REPO))

from paper_1303_2285_b200.workloads import make_input, workload  # noqa: E402

SAMPLE = 4096


def _import_reference():
    src = Path("/root/reference/pkg/src")
    dst = Path("/tmp/covcomb_golden_src")
    if dst.exists():
        shutil.rmtree(dst)
    shutil.copytree(src, dst)
    sys.path.insert(0, str(dst))
    import covcomb  # noqa: F401

    return covcomb


def checksum(packed: np.ndarray) -> np.ndarray:
    """[sum w_k x_k (re, im), ||x||_F, sum re(x_k)] with unit-modulus weights."""
    k = np.arange(packed.size, dtype=np.float64)
    w = np.exp(2j * np.pi * np.modf(k * 0.6180339887498949)[0])
    s = np.sum(w * packed)
    return np.array([s.real, s.imag, np.linalg.norm(packed), packed.real.sum()])


def sample_idx(size: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    if size <= SAMPLE:
        return np.arange(size)
    return np.sort(rng.choice(size, SAMPLE, replace=False))


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg5", action="store_true", help="also sample cfg5 classes (~1 min)")
    args = ap.parse_args()
    cc = _import_reference()
    from covcomb import WindowSpec, InputMatrix
    from covcomb import _numpy_kernels as npk

    threads = len(os.sched_getaffinity(0))
    out = {}

    # --- known answers (test_engine.py:24-32, test_baseline.py:43-45) ------------
    out["ka_single"] = cc.estimate_combinations([[2 + 1j]], WindowSpec(1, 1))[0].packed
    out["ka_ones"] = cc.estimate_naive(np.ones((2, 2)), WindowSpec(1, 1)).packed

    # --- degenerate shapes (test_engine.py:63-70) ------------------------------
    for n, m, p, q in [(1, 1, 1, 1), (5, 1, 2, 1), (1, 6, 1, 3), (4, 4, 4, 4), (7, 5, 1, 1),
                       (3, 2, 3, 2), (20, 20, 8, 8), (12, 11, 4, 3), (10, 9, 3, 3)]:
        seed = n + 10 * m + 100 * p + 1000 * q
        mat = InputMatrix.random(n, m, seed)
        key = f"shape_{n}_{m}_{p}_{q}"
        out[key + "_a"] = mat.array
        out[key + "_naive"] = cc.estimate_naive(mat, WindowSpec(p, q)).packed
        out[key + "_comb"] = cc.estimate_combinations(mat, WindowSpec(p, q))[0].packed

    # --- C4 sweep instances (test_acceptance.py:89-99) -------------------------
    rng = np.random.default_rng(0xA11CE)
    inst = []
    for _ in range(200):
        n = int(rng.integers(1, 25))
        m = int(rng.integers(1, 25))
        p = int(rng.integers(1, n + 1))
        q = int(rng.integers(1, m + 1))
        inst.append((n, m, p, q, int(rng.integers(0, 2**32))))
    c4_params = np.array(inst, dtype=np.int64)
    c4_cs = []
    for i, (n, m, p, q, seed) in enumerate(inst):
        mat = InputMatrix.random(n, m, seed)
        packed = cc.estimate_combinations(mat, WindowSpec(p, q))[0].packed
        c4_cs.append(checksum(packed))
        if p * q <= 64:
            out[f"c4_{i}_packed"] = packed
    out["c4_params"] = c4_params
    out["c4_checksums"] = np.array(c4_cs)

    # --- BASELINE configs --------------------------------------------------------
    def ref_cfg(name):
        w = workload(name)
        a = make_input(w).astype(np.complex128)  # exact up-cast for c64 configs
        t0 = time.perf_counter()
        if w.batch == 1:
            packed = cc.estimate_parallel(a, WindowSpec(w.p, w.q), threads=threads)[0].packed
        else:
            packed = None
        print(f"{name}: reference {time.perf_counter() - t0:.2f}s", flush=True)
        return w, a, packed

    w, a, packed = ref_cfg("cfg1")
    out["cfg1_packed"] = packed
    for name in ("cfg2", "cfg2-c64", "cfg3"):
        w, a, packed = ref_cfg(name)
        idx = sample_idx(packed.size, w.seed + 100)
        key = name.replace("-", "_")
        out[key + "_idx"] = idx
        out[key + "_vals"] = packed[idx]
        out[key + "_checksum"] = checksum(packed)
    # cfg4: first 16 snapshots through estimate_batch; two stored in full
    w = workload("cfg4")
    stack = make_input(w).astype(np.complex128)[:16]
    t0 = time.perf_counter()
    covs = cc.estimate_batch(list(stack), WindowSpec(w.p, w.q), threads=threads)
    print(f"cfg4[:16]: reference {time.perf_counter() - t0:.2f}s", flush=True)
    out["cfg4_checksums"] = np.array([checksum(c.packed) for c in covs])
    out["cfg4_snap0_packed"] = covs[0].packed
    out["cfg4_snap7_packed"] = covs[7].packed

    np.savez(HERE / "golden.npz", **out)
    print("wrote", HERE / "golden.npz", sum(v.nbytes for v in out.values()) / 1e6, "MB")

    if args.cfg5:
        # cfg5: the reference's vectorised class kernel on a stratified class
        # sample; each class's slots are returned in slot order (u-major).
        w = workload("cfg5")
        a = make_input(w)
        classes = cc.unique_combinations(WindowSpec(w.p, w.q))
        pick = np.linspace(0, len(classes) - 1, 24).round().astype(int)
        res = {}
        for ci in pick:
            comb = classes[ci]
            t0 = time.perf_counter()
            sums = npk.class_block_sums(a, comb.dr, comb.dc, w.p, w.q)
            res[f"cls_{ci}"] = np.array([comb.dr, comb.dc])
            res[f"sums_{ci}"] = sums
            print(f"cfg5 class {ci} {comb}: {time.perf_counter() - t0:.2f}s", flush=True)
        res["picked"] = pick
        np.savez(HERE / "golden_cfg5.npz", **res)
        print("wrote golden_cfg5.npz", sum(v.nbytes for v in res.values()) / 1e6, "MB")


if __name__ == "__main__":
    main()
