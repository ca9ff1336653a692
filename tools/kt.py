"""Per-kernel CUDA-event times of one config (development aid)."""
import os, sys
__import__("os").environ.setdefault("COVGPU_TEST_HOOKS", "1")  # COVGPU_* switches are test hooks
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_1303_2285_b200 import WindowSpec
from paper_1303_2285_b200.plan import Plan
from paper_1303_2285_b200.workloads import make_input, workload

for name in sys.argv[1:]:
    w = workload(name)
    dt = torch.complex128 if w.dtype == "c128" else torch.complex64
    plan = Plan(w.n, w.m, WindowSpec(w.p, w.q), batch=w.batch, dtype=dt)
    a = torch.as_tensor(make_input(w), device="cuda").reshape(w.batch, w.n, w.m)
    out = plan.alloc_output()
    for _ in range(2):
        plan.execute(a, out)
    plan.set_timing(True)
    acc = None
    reps = 5
    for _ in range(reps):
        plan.execute(a, out)
        kt = plan.kernel_times()
        acc = kt if acc is None else [x + y for x, y in zip(acc, kt)]
    kt = [x / reps for x in acc]
    names = plan.kernel_names()
    print(f"{name} variant={os.environ.get('COVGPU_BULK_VARIANT','default')}: " +
          " ".join(f"{k}={x:.3f}" for k, x in zip(names, kt)) + f"  total {sum(kt):.3f} ms", flush=True)
