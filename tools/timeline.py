"""%globaltimer timeline of one config-2 tick (needs the -DGPM_TIMELINE build):
    python -m paper_2411_03289_b200.build --variant=timeline -DGPM_TIMELINE
    GPMPPI_LIB=paper_2411_03289_b200/lib/libgpmppi_b200_timeline.so python tools/timeline.py [config2]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.getcwd())
import bench  # noqa: E402
import paper_2411_03289_b200 as G  # noqa: E402
from paper_2411_03289_b200 import _capi as A  # noqa: E402
from paper_2411_03289_b200 import workloads as W  # noqa: E402

w = W.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "config2"]
p, task, x0 = bench.build_planner(w, G)
tl = np.zeros(32)
for rep in range(4):
    p.plan_step(x0, task)
    G.flush_l2(0)
    A.lib().gpmppi_debug_timeline(A.dptr(tl))  # reset
    p.plan_step(x0, task)
    A.lib().gpmppi_debug_timeline(A.dptr(tl))
    t0 = tl[17]
    names = {17: "stage start", 16: "stage end", 1: "rollout first block", 0: "rollout last block end",
             3: "variance first CTA", 2: "variance last CTA end", 5: "reduce first block (after wait)",
             4: "reduce last block end", 9: "tmean after wait", 6: "tmean chain end", 8: "tmean tail end (flag 1)",
             11: "tvar first block", 10: "tvar last block end", 13: "tcov after flag 1", 12: "tightening end (done word)",
             21: "tvar last step: first block go", 20: "tvar last step: last block go",
             18: "recursion step 0 in", 29: "tvar step 0: first block go", 31: "tvar step 0: first block done",
             14: "tvar step 0: last block done", 27: "tvar step 0: cv block starts", 25: "tvar step 0: cv_0 flag raised", 22: "recursion step T/2 in",
             28: "recursion step 3T/4 in", 26: "recursion last step in", 24: "recursion done",
             15: "cv stager: cv_0 staged", 19: "cv stager: cv_T/2 staged", 23: "cv stager: last cv staged"}
    print(f"--- tick {rep}")
    for i in (17, 16, 1, 0, 3, 2, 5, 4, 9, 6, 8, 11, 29, 31, 14, 27, 25, 21, 20, 10, 15, 19, 23, 18, 22, 28, 26, 24, 12):
        print(f"{names[i]:32s} {(tl[i] - t0) / 1e3:9.2f} us")
