"""Quick CUDA-event timing of every config (development aid, not the bench)."""
import sys, time
__import__("os").environ.setdefault("COVGPU_TEST_HOOKS", "1")  # COVGPU_* switches are test hooks
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_1303_2285_b200 import WindowSpec, estimate_tensor, estimate_batch_tensor, um_count
from paper_1303_2285_b200.workloads import make_input, workload

REPS = 5
args = [x for x in sys.argv[1:] if not x.startswith("--reps=")]
for x in sys.argv[1:]:
    if x.startswith("--reps="): REPS = int(x[7:])
for name in args or ["cfg1", "cfg2", "cfg2-c64", "cfg3", "cfg4", "cfg5"]:
    w = workload(name)
    a = torch.as_tensor(make_input(w), device="cuda")
    win = WindowSpec(w.p, w.q)
    f = (lambda: estimate_batch_tensor(a, win)) if w.batch > 1 else (lambda: estimate_tensor(a, win))
    out = f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    reps = REPS
    e0.record()
    for _ in range(reps):
        out = f()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    fl = 8.0 * um_count(w.n, w.m, w.p, w.q) * w.batch
    print(f"{name}: {ms:.3f} ms  {fl/ms/1e9:.2f} TFLOP/s eff  {w.pq**2*w.batch/ms/1e6:.3f} Gentries/s", flush=True)
