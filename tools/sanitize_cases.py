"""Small cases over every kernel family and host path, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck): direct CUDA-core kernels
(cfg1, cfg2), the spectral path (forced, with walk cuts: Q > 16), the tile
finalize in all three layouts, a batched complex64 stack, the host-buffer
paths (sync and async) and the row-band parts.  Prints one line per case."""
import os
__import__("os").environ.setdefault("COVGPU_TEST_HOOKS", "1")  # COVGPU_* switches are test hooks
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1303_2285_b200 import WindowSpec, estimate_combinations  # noqa: E402
from paper_1303_2285_b200.distributed import simulate_rowband  # noqa: E402
from paper_1303_2285_b200.engine import estimate_batch_tensor  # noqa: E402
from paper_1303_2285_b200.plan import Plan  # noqa: E402
from paper_1303_2285_b200.workloads import make_input  # noqa: E402

rng = np.random.default_rng(5)


def rnd(*shape, dt=np.complex128):
    return (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)).astype(dt)


def case(name, fn):
    fn()
    fn()  # the second identical call replays the captured graph
    torch.cuda.synchronize()
    print("case ok:", name, flush=True)


case("cfg1 direct", lambda: estimate_combinations(make_input("cfg1"), WindowSpec(4, 4)))
a2 = make_input("cfg2")
case("cfg2 direct", lambda: estimate_combinations(a2, WindowSpec(16, 16)))

os.environ["COVGPU_SPECTRAL"] = "1"
sp = Plan(96, 80, WindowSpec(12, 10), dtype=torch.complex128)
sp2 = Plan(70, 90, WindowSpec(9, 40), dtype=torch.complex128)  # Q > 16: walk cuts (delta units)
del os.environ["COVGPU_SPECTRAL"]
b1 = torch.as_tensor(rnd(96, 80), device="cuda")
b2 = torch.as_tensor(rnd(70, 90), device="cuda")
for lay in ("dense", "packed", "compact"):
    o1, o2 = sp.alloc_output(lay), sp2.alloc_output(lay)
    case(f"spectral {lay}", lambda: (sp.execute(b1, o1, lay), sp2.execute(b2, o2, lay)))

st = torch.as_tensor(rnd(4, 40, 37, dt=np.complex64), device="cuda")
case("batched c64", lambda: estimate_batch_tensor(st, WindowSpec(7, 5)))
stq = torch.as_tensor(rnd(3, 40, 60, dt=np.complex64), device="cuda")
case("batched c64 Q>16", lambda: estimate_batch_tensor(stq, WindowSpec(6, 20)))

hp = Plan(96, 80, WindowSpec(12, 10), dtype=torch.complex128)
ha = torch.from_numpy(rnd(1, 96, 80)).pin_memory()
hr = torch.empty(hp.output_elems("packed"), dtype=torch.complex128).pin_memory()
case("execute_host", lambda: hp.execute_host(ha, hr, "packed"))
hr2 = torch.empty_like(hr).pin_memory()


def async_pair():
    hp.execute_host_async(ha, hr, "packed")
    hp.execute_host_async(ha, hr2, "packed")
    hp.wait()


case("execute_host_async", async_pair)
os.environ["COVGPU_SPECTRAL"] = "1"
rb = torch.as_tensor(rnd(120, 100), device="cuda")
case("row-band parts x2", lambda: simulate_rowband([rb, rb], WindowSpec(10, 20)))
del os.environ["COVGPU_SPECTRAL"]
print("all cases ok")
