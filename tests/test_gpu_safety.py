"""Memory- and race-safety evidence without compute-sanitizer (closed on
this GPU pool): output guard bands (no write outside the output, every
layout and path), bitwise repeatability under repetition and concurrent
streams (races and uninitialised reads show up as changing bits), and
concurrent executes of one plan on two streams (the plan's workspace is
ordered by its completion event)."""

import os

import numpy as np
import pytest
import torch

from paper_1303_2285_b200 import WindowSpec
from paper_1303_2285_b200.plan import Plan

pytestmark = pytest.mark.gpu

GUARD = 4096
SHAPES = [  # (n, m, p, q, batch, dtype, force spectral)
    (32, 32, 4, 4, 1, torch.complex128, False),
    (96, 80, 12, 10, 1, torch.complex128, True),
    (70, 90, 9, 40, 1, torch.complex128, True),      # walk cuts (Q > 16)
    (40, 37, 7, 5, 4, torch.complex64, False),
    (40, 60, 6, 20, 3, torch.complex64, False),      # batched, walk cuts
    (150, 140, 70, 66, 1, torch.complex128, True),   # P > 64: one stage buffer
    (3, 125, 1, 58, 2, torch.complex128, False),     # P = 1
]


def _plan(n, m, p, q, batch, dt, spectral, cuda):
    if spectral:
        os.environ["COVGPU_SPECTRAL"] = "1"
    try:
        return Plan(n, m, WindowSpec(p, q), batch=batch, dtype=dt, device=cuda)
    finally:
        os.environ.pop("COVGPU_SPECTRAL", None)


def _input(n, m, batch, dt, cuda, seed=3):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((batch, n, m)) + 1j * rng.standard_normal((batch, n, m))
    return torch.as_tensor(a, device=cuda).to(dt)


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("layout", ["dense", "packed", "compact"])
def test_output_guard_bands(cuda, shape, layout):
    """Every kernel writes only inside the output: guard bands of sentinels
    before and after it stay untouched; the result is the same as in an
    unguarded buffer, bit for bit, over repeated executes (graph replay
    included)."""
    n, m, p, q, batch, dt, spectral = shape
    plan = _plan(n, m, p, q, batch, dt, spectral, cuda)
    a = _input(n, m, batch, dt, cuda)
    ne = plan.output_elems(layout)
    sentinel = complex(1.25e300, -3.5e300) if dt == torch.complex128 else complex(1.25e30, -3.5e30)
    buf = torch.full((ne + 2 * GUARD,), sentinel, dtype=dt, device=cuda)
    out = buf[GUARD:GUARD + ne]
    first = None
    for _ in range(4):
        plan.execute(a, out, layout)
        torch.cuda.synchronize()
        assert bool((buf[:GUARD] == sentinel).all()) and bool((buf[GUARD + ne:] == sentinel).all())
        first = out.clone() if first is None else first
        assert torch.equal(out, first)
    plain = plan.alloc_output(layout)
    plan.execute(a, plain, layout)
    assert torch.equal(plain, first)
    plan.close()


@pytest.mark.parametrize("shape", SHAPES[:5])
def test_repeatable_under_concurrent_streams(cuda, shape):
    """Two executes of ONE plan on two different streams back to back, with
    different inputs (the ADVICE race: shared workspace): each result
    equals the same estimate run alone."""
    n, m, p, q, batch, dt, spectral = shape
    plan = _plan(n, m, p, q, batch, dt, spectral, cuda)
    a1, a2 = _input(n, m, batch, dt, cuda, 1), _input(n, m, batch, dt, cuda, 2)
    r1, r2 = plan.alloc_output(), plan.alloc_output()
    plan.execute(a1, r1)
    plan.execute(a2, r2)
    torch.cuda.synchronize()
    ref1, ref2 = r1.clone(), r2.clone()
    s1, s2 = torch.cuda.Stream(cuda), torch.cuda.Stream(cuda)
    for _ in range(5):
        o1, o2 = plan.alloc_output(), plan.alloc_output()
        torch.cuda.synchronize()
        plan.execute(a1, o1, stream=s1)
        plan.execute(a2, o2, stream=s2)
        torch.cuda.synchronize()
        assert torch.equal(o1, ref1) and torch.equal(o2, ref2)
    plan.close()


def test_plan_cache_survives_eviction_under_threads(cuda):
    """More than the cache's 32 shapes from several threads at once: cached
    plans evicted by one thread are never freed under another's execute."""
    import threading

    from paper_1303_2285_b200.engine import estimate_tensor
    from oracle import covoracle as co

    errors = []

    def work(tid):
        try:
            torch.cuda.set_device(cuda)
            rng = np.random.default_rng(tid)
            for k in range(12):
                n, m = 10 + (tid * 12 + k) % 40, 11 + k
                a_np = rng.standard_normal((n, m)) + 1j * rng.standard_normal((n, m))
                got = estimate_tensor(torch.as_tensor(a_np, device=cuda), WindowSpec(3, 2)).cpu().numpy()
                if co.rel_frobenius(got, co.covariance(a_np, 3, 2)) > 1e-12:
                    errors.append((tid, n, m))
        except Exception as exc:  # noqa: BLE001
            errors.append((tid, repr(exc)))

    threads = [threading.Thread(target=work, args=(t,)) for t in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors


def test_env_switches_are_ignored_without_the_test_hook_flag(cuda):
    """The COVGPU_* switches are test hooks: a process without
    COVGPU_TEST_HOOKS=1 takes the product path whatever they say."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    code = (
        "import sys; sys.path.insert(0, %r)\n"
        "import torch\n"
        "from paper_1303_2285_b200 import WindowSpec\n"
        "from paper_1303_2285_b200.plan import Plan\n"
        "p = Plan(64, 64, WindowSpec(4, 8), batch=2, dtype=torch.complex64)\n"
        "q = Plan(300, 300, WindowSpec(8, 8), dtype=torch.complex128)\n"
        "print(p.path, q.path)\n" % str(root)
    )
    env = {k: v for k, v in os.environ.items() if not k.startswith("COVGPU_")}
    env.update({"COVGPU_NO_SNAP": "1", "COVGPU_SPECTRAL": "1"})
    plain = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert plain.returncode == 0, plain.stderr
    hooked = subprocess.run([sys.executable, "-c", code], env={**env, "COVGPU_TEST_HOOKS": "1"},
                            capture_output=True, text=True, timeout=300)
    assert hooked.returncode == 0, hooked.stderr
    snap, small = (int(x) for x in plain.stdout.split())
    assert snap & 8 and not small & 1          # product path: snapshot kernel, direct kernels for the small shape
    snap_h, small_h = (int(x) for x in hooked.stdout.split())
    assert not snap_h & 8 and small_h & 1      # hooks honoured: CUDA-core engine, spectral engine forced
