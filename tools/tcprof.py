"""Per-role cycle breakdown of the tcgen05 variance kernel (GPMPPI_TC_DEBUG=512)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.getcwd())
os.environ.setdefault("GPMPPI_TC_DEBUG", "512")
import paper_2411_03289_b200 as G  # noqa: E402
from paper_2411_03289_b200 import _capi as A  # noqa: E402
from paper_2411_03289_b200 import workloads as W  # noqa: E402
from bench import build_planner  # noqa: E402

w = W.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "config2"]
p, task, x0 = build_planner(w, G, var_path=1)
p.bench_device(x0, task, 2)
out = np.zeros(16)
A.lib().gpmppi_debug_tc_profile(A.dptr(out))
ticks = 5
ms, ph = p.bench_device(x0, task, ticks)
A.lib().gpmppi_debug_tc_profile(A.dptr(out))
ctas = out[11]
names = ["B wait empty_b", "MMA wait tempty", "MMA wait full_a", "MMA wait full_b",
         "A wait empty_a (lane0/warp)", "EPI wait tfull (lane0/warp)", "B total", "MMA total",
         "producers total (per warp)", "epilogue total (per warp)", "-", "-",
         "producer compute+store (per warp)", "MMA issue (excl. waits)", "epilogue drain (per warp)"]
per = {0: ctas, 1: ctas, 2: ctas, 3: ctas, 4: ctas * 8, 5: ctas * 4, 6: ctas, 7: ctas, 8: ctas * 8, 9: ctas * 4,
       10: 1, 11: 1, 12: ctas * 8, 13: ctas, 14: ctas * 4}
print(f"variance phase {ph[1] / ticks * 1e3:.1f} us/tick; CTAs {ctas:.0f}")
for i, nm in enumerate(names):
    if nm == "-":
        continue
    print(f"{nm:32s} {out[i] / per[i] / 1.965e3:9.1f} us per role-instance")
