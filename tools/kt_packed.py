import sys, time
__import__("os").environ.setdefault("COVGPU_TEST_HOOKS", "1")  # COVGPU_* switches are test hooks
sys.path.insert(0, '/root/repo')
import torch
from paper_1303_2285_b200 import WindowSpec
from paper_1303_2285_b200.plan import Plan
from paper_1303_2285_b200.workloads import make_input, workload
for name in sys.argv[1:]:
    w = workload(name)
    dt = torch.complex128 if w.dtype == "c128" else torch.complex64
    plan = Plan(w.n, w.m, WindowSpec(w.p, w.q), batch=w.batch, dtype=dt)
    a = torch.as_tensor(make_input(w), device="cuda").reshape(w.batch, w.n, w.m)
    out = plan.alloc_output("packed")
    for _ in range(3): plan.execute(a, out, "packed")
    plan.set_timing(True)
    acc = None
    for _ in range(5):
        plan.execute(a, out, "packed"); kt = plan.kernel_times(); acc = kt if acc is None else [x+y for x,y in zip(acc, kt)]
    print(name, "packed", " ".join(f"{k}={x/5:.3f}" for k, x in zip(plan.kernel_names(), acc)), f"total {sum(acc)/5:.3f}")
