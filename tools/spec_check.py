"""Spectral core sums vs the tensor-core path (development aid): relF,
per-class worst error, and CUDA-event step / per-kernel times."""
import os, sys
__import__("os").environ.setdefault("COVGPU_TEST_HOOKS", "1")  # COVGPU_* switches are test hooks
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_1303_2285_b200 import WindowSpec
from paper_1303_2285_b200.plan import Plan
from paper_1303_2285_b200.workloads import make_input, workload


def run(plan, a, reps=10):
    out = plan.alloc_output("dense")
    plan.execute(a, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        plan.execute(a, out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    plan.set_timing(True)
    plan.execute(a, out)
    torch.cuda.synchronize()
    kt = {k: round(v, 4) for k, v in plan.kernel_timing().items()}
    plan.set_timing(False)
    return out.clone(), ms, kt


for name in sys.argv[1:] or ["cfg3", "cfg5"]:
    w = workload(name)
    a = torch.as_tensor(make_input(w), device="cuda")
    win = WindowSpec(w.p, w.q)
    os.environ["COVGPU_NO_SPECTRAL"] = "1"
    ref_plan = Plan(w.n, w.m, win, w.batch, a.dtype)
    del os.environ["COVGPU_NO_SPECTRAL"]
    sp_plan = Plan(w.n, w.m, win, w.batch, a.dtype)
    r_ref, ms_ref, kt_ref = run(ref_plan, a)
    r_sp, ms_sp, kt_sp = run(sp_plan, a)
    d = r_sp - r_ref
    relf = (torch.linalg.norm(d) / torch.linalg.norm(r_ref)).item()
    pq = w.p * w.q
    R1, R2 = r_ref.view(-1, pq, pq)[0], r_sp.view(-1, pq, pq)[0]
    # per-diagonal (d = dc*P + dr) worst relative error of the diagonal's entries
    worst = 0.0
    for dd in range(0, pq, max(1, pq // 64)):
        x1, x2 = torch.diagonal(R1, dd), torch.diagonal(R2, dd)
        e = (torch.linalg.norm(x2 - x1) / torch.linalg.norm(x1)).item()
        worst = max(worst, e)
    herm = bool(torch.equal(R2, R2.conj().T))
    print(f"{name}: relF spectral vs tensor-core {relf:.3e}, worst sampled diagonal {worst:.3e}, "
          f"hermitian {herm}")
    print(f"  tensor-core step {ms_ref:.3f} ms  {kt_ref}")
    print(f"  spectral    step {ms_sp:.3f} ms  {kt_sp}")
