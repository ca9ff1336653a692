"""Synchronous host-path time of a workload (dev aid): pinned buffers,
covgpu_plan_execute_host, packed R, median of K calls."""
import sys, time
__import__("os").environ.setdefault("COVGPU_TEST_HOOKS", "1")  # COVGPU_* switches are test hooks
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_1303_2285_b200 import WindowSpec
from paper_1303_2285_b200.plan import Plan
from paper_1303_2285_b200.workloads import make_input, workload

for name in sys.argv[1:] or ["cfg5"]:
    w = workload(name)
    ah = torch.from_numpy(make_input(w)).reshape(w.batch, w.n, w.m).pin_memory()
    plan = Plan(w.n, w.m, WindowSpec(w.p, w.q), w.batch, ah.dtype)
    rh = torch.empty(plan.output_elems("packed"), dtype=ah.dtype).pin_memory()
    ref = torch.empty_like(rh)
    plan.execute_host(ah, ref, "packed")
    ts = []
    for _ in range(10):
        t0 = time.perf_counter()
        plan.execute_host(ah, rh, "packed")
        ts.append(time.perf_counter() - t0)
    ts.sort()
    print(f"{name}: sync e2e median {ts[5]*1e3:.3f} ms min {ts[0]*1e3:.3f} ms; repeat bitwise {torch.equal(rh, ref)}")
    plan.close()
