"""One warm plan execute of a workload (for ncu captures)."""
import sys
__import__("os").environ.setdefault("COVGPU_TEST_HOOKS", "1")  # COVGPU_* switches are test hooks
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_1303_2285_b200 import WindowSpec
from paper_1303_2285_b200.plan import Plan
from paper_1303_2285_b200.workloads import make_input, workload

w = workload(sys.argv[1] if len(sys.argv) > 1 else "cfg5")
a = torch.as_tensor(make_input(w), device="cuda")
plan = Plan(w.n, w.m, WindowSpec(w.p, w.q), w.batch, a.dtype)
out = plan.alloc_output("dense")
for _ in range(2):
    plan.execute(a, out)
torch.cuda.synchronize()
print("ok", plan.kernel_names() if hasattr(plan, "kernel_names") else "")
