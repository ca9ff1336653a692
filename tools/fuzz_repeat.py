"""Re-run the GPU fuzz shapes (test_random_shapes_fuzz) several times and
report every shape whose result differs from the C oracle or between runs
(dev aid for races / uninitialised reads)."""
import os
__import__("os").environ.setdefault("COVGPU_TEST_HOOKS", "1")  # COVGPU_* switches are test hooks
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import covoracle, covoracle_c  # noqa: E402
from paper_1303_2285_b200 import WindowSpec  # noqa: E402
from paper_1303_2285_b200.engine import estimate_batch_tensor  # noqa: E402

spectral = len(sys.argv) > 1 and sys.argv[1] == "1"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
only = int(sys.argv[3]) if len(sys.argv) > 3 else -1
rng = np.random.default_rng(20261020 + (7 if spectral else 0))
if spectral:
    os.environ["COVGPU_SPECTRAL"] = "1"
bad = 0
for it in range(60):
    n = int(rng.integers(1, 160))
    m = int(rng.integers(1, 160))
    p = int(rng.integers(1, min(n, 70) + 1))
    q = int(rng.integers(1, min(m, 70) + 1))
    batch = int(rng.integers(1, 4))
    dt = np.complex128 if it % 2 == 0 else np.complex64
    stack = (rng.standard_normal((batch, n, m)) + 1j * rng.standard_normal((batch, n, m))).astype(dt)
    if only >= 0 and it != only:
        continue
    k = (n - p + 1) * (m - q + 1)
    refs = [covoracle_c.estimate_packed(stack[b].astype(np.complex128), p, q) / k for b in range(batch)]
    first = None
    for r in range(reps):
        try:
            got = estimate_batch_tensor(stack, WindowSpec(p, q)).cpu().numpy()
        except RuntimeError as exc:
            print(f"it={it} n={n} m={m} p={p} q={q} B={batch} dt={dt.__name__}: {exc}", flush=True)
            bad += 1
            break
        if first is None:
            first = got
        same = np.array_equal(first, got)
        for b in range(batch):
            iu = np.triu_indices(p * q)
            err = covoracle.rel_frobenius(got[b].astype(np.complex128)[iu], refs[b])
            tol = 1e-12 if dt == np.complex128 else 1e-5
            if err > tol or not same:
                bad += 1
                d = np.abs(got[b].astype(np.complex128)[iu] - refs[b])
                worst = np.unravel_index(np.argmax(np.abs(got[b] - (first[b]))), got[b].shape) if not same else None
                print(f"it={it} rep={r} n={n} m={m} p={p} q={q} B={batch} dt={dt.__name__} b={b} "
                      f"relF={err:.3e} same_as_first={same} maxabs={d.max():.3e} worst_diff_at={worst}", flush=True)
print("bad", bad)
