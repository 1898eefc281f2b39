"""Build the config-2 planner, run warm ticks, then exactly one more tick (for ncu captures:
--launch-skip 6*WARM --launch-count 6 selects the last tick's six kernels)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2411_03289_b200 as G  # noqa: E402
from paper_2411_03289_b200 import workloads as W  # noqa: E402
w = W.CONFIGS[os.environ.get("CFG", "config2")]
p, task, x0 = bench.build_planner(w, G)
for _ in range(int(os.environ.get("WARM", "3"))):
    p.plan_step(x0, task)
G.flush_l2(0)
p.plan_step(x0, task)
print("one tick done")
