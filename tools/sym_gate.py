"""Step time with and without the symmetric core sums on mid-size shapes (dev aid)."""
import os, sys
from pathlib import Path
os.environ.setdefault("COVGPU_TEST_HOOKS", "1")
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_1303_2285_b200 import WindowSpec
from paper_1303_2285_b200.plan import Plan

def step(n, m, p, q, env):
    for k, v in env.items(): os.environ[k] = v
    try:
        plan = Plan(n, m, WindowSpec(p, q), dtype=torch.complex128)
    finally:
        for k in env: del os.environ[k]
    rng = np.random.default_rng(1)
    a = torch.as_tensor(rng.standard_normal((1, n, m)) + 1j * rng.standard_normal((1, n, m)), device="cuda")
    out = plan.alloc_output()
    flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
    for _ in range(3): plan.execute(a, out)
    ts = []
    for _ in range(15):
        flush.fill_(1); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); plan.execute(a, out); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    plan.close()
    return sorted(ts)[7]

for shp in [(512, 512, 32, 32), (1024, 1024, 32, 32), (1024, 1024, 64, 64), (1500, 900, 40, 50), (1536, 1536, 64, 64), (4096, 512, 64, 64), (2048, 2048, 16, 16)]:
    t0 = step(*shp, {"COVGPU_NO_SYM": "1", "COVGPU_SPECTRAL": "1"})
    t1 = step(*shp, {"COVGPU_SYM": "1", "COVGPU_SPECTRAL": "1"})
    print(shp, f"two-mask {t0:.4f} ms, symmetric {t1:.4f} ms", flush=True)
