"""Small workload touching every device kernel once, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck; tools/sanitize.sh)."""
import dataclasses
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_03289_b200 as G  # noqa: E402
from paper_2411_03289_b200 import harness as H  # noqa: E402
from paper_2411_03289_b200 import workloads as W  # noqa: E402

w = dataclasses.replace(W.CONFIGS["config2"], samples=300, horizon=12, n_points=96, n_obstacles=4)
X, Y, Kp = W.gp_training_set(w.n_points, 3, seed=1)
gp = G.GpModel.fit(X, Y, Kp)
task, _, obs = W.make_task_objects(w, G)
x0 = np.array(w.x0)
for vp in (0, 1, 3):  # FFMA, 3xTF32, 3xFP16 variance kernels + rollout / reduce / tightening
    p = G.Planner(G.MppiConfig(samples=w.samples, horizon=w.horizon, seed=3), G.GpEnsemble(gp, 3))
    p.set_variance_path(vp)
    for t in range(2):
        p.plan_step(x0, task)
    p.set_command_first(True)
    p.plan_step(x0, task)
    p.wait_tightening()
    p.inject_noise(p.philox_noise(0))
    p.plan_step(x0, task)
    p.sample_weights(), p.flags(), p.lane_radii(), p.obstacle_margins()
p.set_noise_mode(G.NOISE_PHILOX)
p.set_shard(0, w.samples)
p.attach_comm(G.nccl_unique_id(), 1, 0)  # ncclAllGather + finish_kernel
p.plan_step(x0, task)
for kind in (G.NominalDynamic(), G.UnicycleBaseline()):  # rollout_base_kernel
    q = G.Planner(G.MppiConfig(samples=200, horizon=10), kind)
    q.plan_step(x0, task)
bp = G.BatchPlanner(G.MppiConfig(samples=128, horizon=10), G.GpEnsemble(gp, 3), 3)
bp.plan_step(np.tile(x0, (3, 1)), [task] * 3)
gp.predict_batch(X[:7] + 0.01)  # predict_kernel
for path in (0, 1, 2, 3):
    gp.variance_batch(X[:200], path)
G.rollout(x0, np.zeros((8, 2)), G.GpEnsemble(gp, 3), [1 / 3] * 3)  # free functions
e = G.sample_perturbations(G.MppiConfig(samples=16, horizon=8), 0)
wts = G.trajectory_weights(np.linspace(0.0, 1.0, 16), 0.1)
G.update_controls(np.zeros((8, 2)), e, wts)
G.shift_horizon(np.zeros((8, 2)))
os.environ["GPMPPI_FIT"] = "device"
G.GpModel.fit(X[:40], Y[:40], Kp)  # fit.cu Cholesky + inverse
H.select_kernel_grid(X[:24], Y[:24, :2])  # fit.cu grid kernel
print("sanitize workload done")
