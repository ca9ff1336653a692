"""Timeline of one device-path step (CUPTI via torch.profiler): every kernel of
the plan's three streams with start / end relative to the first (dev aid)."""
import sys
from pathlib import Path
__import__("os").environ.setdefault("COVGPU_TEST_HOOKS", "1")
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from torch.profiler import ProfilerActivity, profile
from paper_1303_2285_b200 import WindowSpec
from paper_1303_2285_b200.plan import Plan
from paper_1303_2285_b200.workloads import make_input, workload

w = workload(sys.argv[1] if len(sys.argv) > 1 else "cfg5")
a = torch.as_tensor(make_input(w), device="cuda")
plan = Plan(w.n, w.m, WindowSpec(w.p, w.q), w.batch, a.dtype)
out = plan.alloc_output("dense")
flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
for _ in range(4):
    plan.execute(a, out)
flush.fill_(1)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    plan.execute(a, out)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start
for e in evs:
    s, d = (e.time_range.start - t0) / 1e3, (e.time_range.end - e.time_range.start) / 1e3
    print(f"{s:8.4f} -> {s + d:8.4f} ms ({d*1e3:6.1f} us)  {e.name[:70]}")
