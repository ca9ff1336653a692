"""K2 (snap.cuh) against the C oracle and the CUDA-core path (dev aid)."""
import os, sys
__import__("os").environ.setdefault("COVGPU_TEST_HOOKS", "1")  # COVGPU_* switches are test hooks
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from oracle import covoracle
from oracle import covoracle_c
from paper_1303_2285_b200 import WindowSpec
from paper_1303_2285_b200.plan import Plan

shapes = [(128, 128, 8, 16, 6), (96, 100, 5, 9, 3), (64, 128, 8, 2, 2), (40, 37, 2, 16, 3), (128, 77, 7, 12, 4)]
for n, m, p, q, batch in shapes:
    rng = np.random.default_rng(n * 1000 + m)
    a = (rng.standard_normal((batch, n, m)) + 1j * rng.standard_normal((batch, n, m))).astype(np.complex64)
    ad = torch.as_tensor(a, device="cuda")
    win = WindowSpec(p, q)
    plan = Plan(n, m, win, batch=batch, dtype=torch.complex64)
    out = plan.alloc_output("dense")
    plan.execute(ad, out)
    got = out.reshape(batch, p * q, p * q).cpu().numpy()
    os.environ["COVGPU_NO_SNAP"] = "1"
    plan0 = Plan(n, m, win, batch=batch, dtype=torch.complex64)
    del os.environ["COVGPU_NO_SNAP"]
    out0 = plan0.alloc_output("dense")
    plan0.execute(ad, out0)
    got0 = out0.reshape(batch, p * q, p * q).cpu().numpy()
    worst = worst0 = 0.0
    for b in range(batch):
        ref = covoracle.covariance(a[b].astype(np.complex128), p, q)
        worst = max(worst, covoracle.rel_frobenius(got[b], ref))
        worst0 = max(worst0, covoracle.rel_frobenius(got0[b], ref))
    herm = bool(np.array_equal(got, got.conj().transpose(0, 2, 1)))
    print(f"{n}x{m} P={p} Q={q} B={batch}: path {plan.path} relF snap {worst:.2e} (cuda-core {worst0:.2e}) hermitian {herm}", flush=True)
