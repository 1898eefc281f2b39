"""Synthetic workloads of BASELINE.json's configs.

GP: n inputs uniform in the command box v, v_ref ∈ [-0.5, 2], ω, ω_ref ∈ [-2, 2]
(test_gp.cpp:15-22); 2R outputs y_{2t} = 0.02 sin(x0 + t) + 0.01 x2,
y_{2t+1} = -0.015 x3 + 0.005 t (test_mppi.cpp:189-192); one shared kernel
sf2 = 4e-3, l = (0.8, 1.2, 0.8, 1.2), sn2 = 1e-4 (test_harness.cpp:21-24).
Obstacles: random_obstacle_field (harness.cpp:120-144) with the config.hpp:57-63
box. Synthetic data, random GP of the named shape (no datasets).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

KERNEL = (4e-3, 0.8, 1.2, 0.8, 1.2, 1e-4)


def gp_training_set(n: int, R: int, seed: int = 0):
    rng = np.random.default_rng(seed)
    x = np.column_stack([rng.uniform(-0.5, 2.0, n), rng.uniform(-2, 2, n),
                         rng.uniform(-0.5, 2.0, n), rng.uniform(-2, 2, n)])
    y = np.empty((n, 2 * R))
    for t in range(R):
        y[:, 2 * t] = 0.02 * np.sin(x[:, 0] + t) + 0.01 * x[:, 2]
        y[:, 2 * t + 1] = -0.015 * x[:, 3] + 0.005 * t
    kernels = np.tile(np.array(KERNEL), (2 * R, 1))
    return x, y, kernels


def random_obstacle_field(count: int, seed: int, start=(0.0, 0.0), goal=(8.0, 0.0),
                          capture=0.5, x_range=(1.5, 6.5), y_range=(-2.5, 2.5),
                          r_range=(0.25, 0.5), min_gap=0.5):
    """Rejection sampling as harness.cpp:120-144 (numpy RNG stream)."""
    rng = np.random.default_rng(seed)
    out = []
    attempts = 0
    while len(out) < count:
        attempts += 1
        if attempts > 10000:
            raise RuntimeError("random_obstacle_field: rejection sampling exceeded 10000 attempts")
        c = np.array([rng.uniform(*x_range), rng.uniform(*y_range)])
        r = rng.uniform(*r_range)
        if np.hypot(*(c - np.asarray(start))) < r + min_gap:
            continue
        if np.hypot(*(c - np.asarray(goal))) < r + capture + min_gap:
            continue
        out.append([c[0], c[1], r])
    return np.array(out).reshape(-1, 3)


@dataclass
class Workload:
    name: str
    samples: int
    horizon: int
    n_points: int  # 0 → GP-free model
    terrains: int
    task: str  # tracking | avoidance | combined
    track: str  # circle | lane
    n_obstacles: int
    x0: tuple
    v_desired: float = 2.0
    p_x: float = 0.95
    model: str = "gp"  # gp | nominal | unicycle | edd5
    lam: float = 0.1
    sigma_sim: tuple = (0.09, 0.25)
    seed: int = 11  # planner seed (acceptance.cpp:430)
    robots: int = 1  # independent planners sharing the model (config 4)

    @property
    def sample_steps(self) -> int:
        return self.robots * self.samples * self.horizon

    def flops_per_sample_step(self) -> int:
        """F = n² + 24n algorithmic FLOP per sample-rollout-step."""
        n = self.n_points
        return n * n + 24 * n


CONFIGS = {
    # configs[0]: nominal dynamic unicycle, no GP, path following
    "config1": Workload("config1", 1024, 40, 0, 1, "tracking", "circle", 0,
                        (2.0, 0.0, np.pi / 2, 0.0, 0.0), model="nominal"),
    # configs[1]: the headline — GP-MPPI path following + 10 tightened obstacles
    "config2": Workload("config2", 4096, 40, 512, 3, "combined", "lane", 10,
                        (0.0, 0.0, 0.0, 0.0, 0.0)),
    # configs[2]: multi-terrain, GP-variance heavy
    "config3": Workload("config3", 16384, 60, 2048, 3, "tracking", "circle", 0,
                        (2.0, 0.0, np.pi / 2, 0.0, 0.0)),
    # configs[3]: 256 independent robots sharing one GP model, one solve each per launch
    "config4": Workload("config4", 4096, 40, 512, 3, "combined", "lane", 10,
                        (0.0, 0.0, 0.0, 0.0, 0.0), robots=256),
    # configs[4] unit: K per GPU in the sharded sweep
    "config5": Workload("config5", 65536, 40, 512, 3, "combined", "lane", 10,
                        (0.0, 0.0, 0.0, 0.0, 0.0)),
}


def make_task_objects(w: Workload, api):
    """Build (task, track, obstacles) with the given API module (product or test mirror)."""
    if w.track == "circle":
        track = api.Track.circle_track((0.0, 0.0), 2.0, 0.4)
    else:
        track = api.Track.polyline_track([[0.0, 0.0], [60.0, 0.0]], 0.4, False)
    obstacles = random_obstacle_field(w.n_obstacles, seed=3) if w.n_obstacles else np.zeros((0, 3))
    if w.task == "tracking":
        task = api.TrackingTask(track, w.v_desired)
    elif w.task == "combined":
        task = api.CombinedTask(track, w.v_desired, obstacles)
    else:
        task = api.AvoidanceTask(obstacles, api.GoalSpec((8.0, 0.0), 0.5))
    return task, track, obstacles


def make_batch_tasks(w: Workload, api):
    """Config 4 scenarios: robot b gets its own obstacle field (seed 3 + b) and a
    lateral start offset; the track, weights and goal are shared."""
    if w.track == "circle":
        track = api.Track.circle_track((0.0, 0.0), 2.0, 0.4)
    else:
        track = api.Track.polyline_track([[0.0, 0.0], [60.0, 0.0]], 0.4, False)
    tasks, x0 = [], np.zeros((w.robots, 5))
    for b in range(w.robots):
        obstacles = random_obstacle_field(w.n_obstacles, seed=3 + b) if w.n_obstacles else np.zeros((0, 3))
        if w.task == "tracking":
            tasks.append(api.TrackingTask(track, w.v_desired))
        elif w.task == "combined":
            tasks.append(api.CombinedTask(track, w.v_desired, obstacles))
        else:
            tasks.append(api.AvoidanceTask(obstacles, api.GoalSpec((8.0, 0.0), 0.5)))
        x0[b] = w.x0
        x0[b, 1] += 0.1 * ((b % 5) - 2) / 2.0
    return tasks, x0
