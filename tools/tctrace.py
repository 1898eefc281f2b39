"""CTA-0 timeline of the tcgen05 variance kernel (GPMPPI_TC_DEBUG bit 4096)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.getcwd())
# the GPMPPI_TC_DEBUG switches exist only in the diagnostics build:
#   python -m paper_2411_03289_b200.build --variant=diag -DGPM_TC_DIAG
os.environ.setdefault("GPMPPI_LIB", os.path.join(os.getcwd(), "paper_2411_03289_b200", "lib", "libgpmppi_b200_diag.so"))
os.environ["GPMPPI_TC_DEBUG"] = str(4096 | int(os.environ.get("TC_EXTRA", "0")))
import paper_2411_03289_b200 as G  # noqa: E402
from paper_2411_03289_b200 import _capi as A  # noqa: E402
from paper_2411_03289_b200 import workloads as W  # noqa: E402
from bench import build_planner  # noqa: E402

w = W.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "config2"]
p, task, x0 = build_planner(w, G, var_path=int(os.environ.get("VAR_PATH", "3")))
p.bench_device(x0, task, 3)
t = np.zeros(64)
A.lib().gpmppi_debug_tc_trace(A.dptr(t))
t0 = t[0]
rel = lambda i: (t[i] - t0) if t[i] else float("nan")  # noqa: E731
print(f"prologue done {rel(1):9.0f}")
for k in range(10):
    print(f"tile {k}: B start {rel(48 + k):9.0f}  A start {rel(36 + k):9.0f}  MMA start {rel(2 + 2 * k):9.0f}"
          f"  tfull commit {rel(3 + 2 * k):9.0f}  epi wake {rel(24 + k):9.0f}")
print(f"MMA end {rel(60):9.0f} epi end {rel(61):9.0f} producer end {rel(62):9.0f} dealloc {rel(63):9.0f}")
print("epilogue done (passes 0-3):", [f"{rel(i):.0f}" for i in (22, 23, 34, 35)])
