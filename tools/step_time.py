"""CUDA-event step time of a workload with the default plan (overlapped
streams, no per-kernel timing), L2 flushed between steps (dev aid)."""
import sys
__import__("os").environ.setdefault("COVGPU_TEST_HOOKS", "1")  # COVGPU_* switches are test hooks
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_1303_2285_b200 import WindowSpec
from paper_1303_2285_b200.plan import Plan
from paper_1303_2285_b200.workloads import make_input, workload

for name in sys.argv[1:] or ["cfg5"]:
    w = workload(name)
    a = torch.as_tensor(make_input(w), device="cuda")
    plan = Plan(w.n, w.m, WindowSpec(w.p, w.q), w.batch, a.dtype)
    lay = __import__("os").environ.get("STEP_LAYOUT", "dense")
    out = plan.alloc_output(lay)
    flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
    for _ in range(3):
        plan.execute(a, out, lay)
    ts = []
    for _ in range(20):
        flush.fill_(1)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); plan.execute(a, out, lay); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    plan.set_timing(True); plan.execute(a, out, lay); torch.cuda.synchronize()
    print(f"{name}: step median {ts[len(ts)//2]:.4f} ms min {ts[0]:.4f} path={plan.path} kernels "
          f"{ {k: round(v, 4) for k, v in plan.kernel_timing().items()} }", flush=True)
    plan.close()
