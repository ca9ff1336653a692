"""Distribution of back-to-back synchronous host-path call times (dev aid)."""
import sys, time
from pathlib import Path
__import__("os").environ.setdefault("COVGPU_TEST_HOOKS", "1")
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_1303_2285_b200 import WindowSpec
from paper_1303_2285_b200.plan import Plan
from paper_1303_2285_b200.workloads import make_input, workload

w = workload(sys.argv[1] if len(sys.argv) > 1 else "cfg5")
ah = torch.from_numpy(make_input(w)).reshape(w.batch, w.n, w.m).pin_memory()
plan = Plan(w.n, w.m, WindowSpec(w.p, w.q), w.batch, ah.dtype)
rh = torch.empty(plan.output_elems("packed"), dtype=ah.dtype).pin_memory()
plan.execute_host(ah, rh, "packed")
ts = []
t00 = time.perf_counter()
for _ in range(30):
    t0 = time.perf_counter()
    plan.execute_host(ah, rh, "packed")
    ts.append((time.perf_counter() - t0) * 1e3)
tot = (time.perf_counter() - t00) * 1e3 / 30
print("mean of loop", round(tot, 3), "calls:", " ".join(f"{t:.2f}" for t in ts))
