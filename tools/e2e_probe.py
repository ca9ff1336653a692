"""Which earlier use of a plan changes the synchronous host-path time (dev aid)."""
import sys, time
__import__("os").environ.setdefault("COVGPU_TEST_HOOKS", "1")  # COVGPU_* switches are test hooks
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_1303_2285_b200 import WindowSpec
from paper_1303_2285_b200.plan import Plan
from paper_1303_2285_b200.workloads import make_input, workload

w = workload(sys.argv[1] if len(sys.argv) > 1 else "cfg5")
ah = torch.from_numpy(make_input(w)).reshape(w.batch, w.n, w.m).pin_memory()
plan = Plan(w.n, w.m, WindowSpec(w.p, w.q), w.batch, ah.dtype)
rh = torch.empty(plan.output_elems("packed"), dtype=ah.dtype).pin_memory()


def e2e(tag):
    plan.execute_host(ah, rh, "packed")
    ts = []
    for _ in range(10):
        t0 = time.perf_counter()
        plan.execute_host(ah, rh, "packed")
        ts.append(time.perf_counter() - t0)
    ts.sort()
    print(f"{tag}: median {ts[5]*1e3:.3f} ms min {ts[0]*1e3:.3f} max {ts[-1]*1e3:.3f}", flush=True)


e2e("fresh plan")
a = ah.cuda()
out = plan.alloc_output("dense")
for _ in range(5):
    plan.execute(a, out, "dense")
torch.cuda.synchronize()
e2e("after 5 device executes (dense)")
plan.set_timing(True)
plan.execute(a, out, "dense")
plan.kernel_times()
plan.set_timing(False)
e2e("after a timing-mode execute")
flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
flush.fill_(1)
torch.cuda.synchronize()
e2e("after a 256 MiB flush buffer")
p2 = Plan(w.n, w.m, WindowSpec(w.p, w.q), w.batch, ah.dtype)
o2 = p2.alloc_output("packed")
p2.execute(a, o2, "packed")
torch.cuda.synchronize()
p2.close()
e2e("after a second plan of the shape came and went")
