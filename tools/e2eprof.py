"""Host-overhead split of the public plan_step at a bench config: Python wall time per
call vs the C-side plan_ms / command_ms (diagnostics) and the device tick (events).
Usage: python tools/e2eprof.py [config2] (GPU required)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.getcwd())
import paper_2411_03289_b200 as G  # noqa: E402
from bench import build_planner  # noqa: E402
from paper_2411_03289_b200 import workloads as W  # noqa: E402

w = W.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "config2"]
p, task, x0 = build_planner(w, G)
d = G.StepDiagnostics()
for _ in range(20):
    p.plan_step(x0, task, d)
py, plan, cmd = [], [], []
for _ in range(300):
    t0 = time.perf_counter()
    p.plan_step(x0, task, d)
    py.append((time.perf_counter() - t0) * 1e3)
    plan.append(d.plan_ms)
    cmd.append(d.command_ms)
dev, _ = p.bench_device(x0, task, 50, flush_l2=False)
print(f"python wall p50 {np.median(py):.4f} ms | C plan_ms p50 {np.median(plan):.4f} | C command_ms p50 "
      f"{np.median(cmd):.4f} | device tick {np.median(dev) if hasattr(dev, '__len__') else dev}")
