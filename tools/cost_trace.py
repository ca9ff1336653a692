"""Measured per-class GPU cost trace (engine.measure_combination_times: every
class alone as a one-class plan, CUDA events, best of 3) written in the
reference's task_id,dr,dc,cost format, plus its rank correlation with the
reference's cost model mu = pair_count (and mu (1 + eta), engine.py:86-92).
Usage: python tools/cost_trace.py cfg3 profiles/r02_cost_trace_cfg3.csv"""
import json
__import__("os").environ.setdefault("COVGPU_TEST_HOOKS", "1")  # COVGPU_* switches are test hooks
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1303_2285_b200 import WindowSpec  # noqa: E402
from paper_1303_2285_b200.combinations import max_writes, pair_count  # noqa: E402
from paper_1303_2285_b200.engine import measure_combination_times, write_cost_trace  # noqa: E402
from paper_1303_2285_b200.workloads import make_input, workload  # noqa: E402


def ranks(x):
    order = np.argsort(x, kind="stable")
    r = np.empty(len(x))
    r[order] = np.arange(len(x))
    return r


w = workload(sys.argv[1])
out = Path(sys.argv[2])
win = WindowSpec(w.p, w.q)
entries = measure_combination_times(make_input(w)[0] if w.batch > 1 else make_input(w), win)
write_cost_trace(out, entries)
cost = np.array([c for _, c in entries])
mu = np.array([pair_count(cb, w.n, w.m) for cb, _ in entries], dtype=float)
model = np.array([pair_count(cb, w.n, w.m) * (1 + max_writes(cb, win)) for cb, _ in entries], dtype=float)
summary = {
    "workload": w.name, "classes": len(entries), "seconds_total": float(cost.sum()),
    "cost_min_us": float(cost.min() * 1e6), "cost_max_us": float(cost.max() * 1e6),
    "spearman_cost_vs_mu": float(np.corrcoef(ranks(cost), ranks(mu))[0, 1]),
    "spearman_cost_vs_mu_1_plus_eta": float(np.corrcoef(ranks(cost), ranks(model))[0, 1]),
    "trace": str(out),
}
out.with_suffix(".json").write_text(json.dumps(summary, indent=1) + "\n")
print(json.dumps(summary))
