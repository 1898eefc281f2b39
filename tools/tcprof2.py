"""Per-role cycle breakdown of the CTA-pair variance kernel (GPMPPI_TC_DEBUG=512, path 4)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.getcwd())
# the GPMPPI_TC_DEBUG switches exist only in the diagnostics build:
#   python -m paper_2411_03289_b200.build --variant=diag -DGPM_TC_DIAG
os.environ.setdefault("GPMPPI_LIB", os.path.join(os.getcwd(), "paper_2411_03289_b200", "lib", "libgpmppi_b200_diag.so"))
os.environ.setdefault("GPMPPI_TC_DEBUG", "512")
import paper_2411_03289_b200 as G  # noqa: E402
from paper_2411_03289_b200 import _capi as A  # noqa: E402
from paper_2411_03289_b200 import workloads as W  # noqa: E402
from bench import build_planner  # noqa: E402

w = W.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "config2"]
p, task, x0 = build_planner(w, G, var_path=4)
p.bench_device(x0, task, 2)
out = np.zeros(16)
A.lib().gpmppi_debug_tc_profile(A.dptr(out))
ticks = 5
ms, ph = p.bench_device(x0, task, ticks)
A.lib().gpmppi_debug_tc_profile(A.dptr(out))
ctas = out[11]
names = {0: ("B wait empty", ctas), 1: ("MMA wait tempty (leader)", ctas / 2), 2: ("MMA wait full (leader)", ctas / 2),
         4: ("A wait empty (lane0/warp)", ctas * 8), 5: ("EPI wait tfull (lane0/warp)", ctas * 4),
         6: ("B total", ctas), 7: ("MMA total (leader)", ctas / 2), 8: ("producers total (per warp)", ctas * 8),
         9: ("epilogue total (per warp)", ctas * 4), 12: ("relay wait full (peer)", ctas / 2),
         13: ("relay total (peer)", ctas / 2)}
print(f"variance phase {ph[1] / ticks * 1e3:.1f} us/tick; CTAs {ctas:.0f}")
for i, (nm, per) in names.items():
    print(f"{nm:32s} {out[i] / per / 1.965e3:9.1f} us per role-instance")
