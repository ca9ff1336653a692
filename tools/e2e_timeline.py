"""Timeline of one synchronous host-path call (CUPTI via torch.profiler): every
memcpy and kernel with start / duration, relative to the first event (dev aid)."""
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
ah = torch.from_numpy(make_input(w)).reshape(w.batch, w.n, w.m).pin_memory()
plan = Plan(w.n, w.m, WindowSpec(w.p, w.q), w.batch, ah.dtype)
rh = torch.empty(plan.output_elems("packed"), dtype=ah.dtype).pin_memory()
for _ in range(3):
    plan.execute_host(ah, rh, "packed")
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    plan.execute_host(ah, rh, "packed")
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start
merged = []
for e in evs:
    name = e.name.split("(")[0][:48]
    s, d = (e.time_range.start - t0) / 1e3, (e.time_range.end - e.time_range.start) / 1e3
    if merged and merged[-1][0] == name and s - merged[-1][2] < 0.02:
        merged[-1][2] = s + d
        merged[-1][3] += 1
    else:
        merged.append([name, s, s + d, 1])
for name, s, e, n in merged:
    print(f"{s:8.3f} -> {e:8.3f} ms  x{n:<4d} {name}")
