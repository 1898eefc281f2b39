"""Debug driver for the co-resident variance: python tools/coopdbg.py <task> <noise> [K]"""
import sys, os, numpy as np, dataclasses
sys.path.insert(0, os.getcwd())
import paper_2411_03289_b200 as G
from paper_2411_03289_b200 import workloads as W
task_kind, noise = sys.argv[1], sys.argv[2]
K = int(sys.argv[3]) if len(sys.argv) > 3 else 512
track = os.environ.get("DBG_TRACK", "lane" if task_kind != "tracking" else "circle")
x0 = (2.0, 0.0, np.pi / 2, 0.0, 0.0) if track == "circle" else (0.0, 0.0, 0.0, 0.0, 0.0)
w = dataclasses.replace(W.CONFIGS["config2"], samples=K, task=task_kind, track=track, x0=x0,
                        n_obstacles=int(os.environ.get("DBG_OBS", "10")))
X, Y, Kp = W.gp_training_set(512, 3, seed=0)
gp = G.GpModel.fit(X, Y, Kp)
p = G.Planner(G.MppiConfig(samples=K, horizon=40, seed=11), G.GpEnsemble(gp, 3))
task = W.make_task_objects(w, G)[0]
for t in range(3):
    if noise == "inj":
        rng = np.random.default_rng(t)
        p.inject_noise(rng.normal(size=(K, 40, 2)) * np.array([0.3, 0.5]))
    print(task_kind, noise, t, p.plan_step(np.array(w.x0), task), flush=True)
