"""Edge cases of the solve path vs the FP64 oracle (same injected reference noise).

Shapes the reference's own suites exercise or that stress the device tiling:
K = 1 / T = 1 / a one-point GP, ragged n (not a multiple of the 16-point chunk),
two distinct kernel groups, one terrain, the maximum obstacle count, a closed
square track, horizons beyond 64 steps (several flag words), and K*T leaving a
lone 128-query tile for the two-tile variance iteration. Tolerances: tests/helpers.py.
"""
import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import SEQ_ATOL, TIGHT_RTOL, assert_tick_parity

pytestmark = pytest.mark.gpu


def _gp_data(n, R, seed, split_kernels=False):
    rng = np.random.default_rng(seed)
    x = np.column_stack([rng.uniform(-0.5, 2.0, n), rng.uniform(-2, 2, n),
                         rng.uniform(-0.5, 2.0, n), rng.uniform(-2, 2, n)])
    y = np.empty((n, 2 * R))
    for t in range(R):
        y[:, 2 * t] = 0.02 * np.sin(x[:, 0] + t) + 0.01 * x[:, 2]
        y[:, 2 * t + 1] = -0.015 * x[:, 3] + 0.005 * t
    k_v = (4e-3, 0.8, 1.2, 0.8, 1.2, 1e-4)
    k_w = (3e-3, 1.0, 1.0, 0.9, 1.1, 2e-4) if split_kernels else k_v
    kernels = np.array([k_v if o % 2 == 0 else k_w for o in range(2 * R)])
    return x, y, kernels


def _tasks(G, kind, track, obstacles):
    if track == "circle":
        td = G.Track.circle_track((0.0, 0.0), 2.0, 0.4)
        to = O.make_track("circle", (0.0, 0.0), 2.0, 0.4)
    elif track == "square":
        pts = [[-2.0, -2.0], [2.0, -2.0], [2.0, 2.0], [-2.0, 2.0]]
        td = G.Track.polyline_track(pts, 0.4, True)
        to = O.make_track("poly", half_width=0.4, waypoints=pts, closed=True)
    else:
        pts = [[0.0, 0.0], [60.0, 0.0]]
        td = G.Track.polyline_track(pts, 0.4, False)
        to = O.make_track("poly", half_width=0.4, waypoints=pts, closed=False)
    if kind == "tracking":
        return G.TrackingTask(td, 1.5), O.make_task(O.ORC_TASK_TRACKING, to, 1.5)
    if kind == "combined":
        return (G.CombinedTask(td, 1.5, obstacles),
                O.make_task(O.ORC_TASK_COMBINED, to, 1.5, obstacles=obstacles if len(obstacles) else None))
    return (G.AvoidanceTask(obstacles, G.GoalSpec((8.0, 0.0), 0.5)),
            O.make_task(O.ORC_TASK_AVOIDANCE, None, 1.5, obstacles=obstacles, goal=(8.0, 0.0, 0.5)))


def _obstacles(count, seed):
    rng = np.random.default_rng(seed)
    return np.column_stack([rng.uniform(0.5, 7.0, count), rng.uniform(-2.5, 2.5, count),
                            rng.uniform(0.1, 0.3, count)]) if count else np.zeros((0, 3))


CASES = {
    # name: (K, T, n, R, task, track, obstacles, split_kernels, x0)
    "K1_T1_n1": (1, 1, 1, 1, "tracking", "circle", 0, False, (2.0, 0.0, np.pi / 2, 0.0, 0.0)),
    "ragged_n17_K33": (33, 3, 17, 3, "avoidance", "lane", 5, False, (0.0, 0.0, 0.0, 0.3, 0.0)),
    "two_kernel_groups": (300, 12, 96, 2, "combined", "lane", 6, True, (0.0, 0.1, 0.0, 0.5, 0.0)),
    "one_terrain_square": (257, 20, 64, 1, "tracking", "square", 0, False, (-2.0, -2.0, 0.0, 0.5, 0.0)),
    "max_obstacles": (200, 10, 48, 3, "combined", "lane", 64, False, (0.0, 0.0, 0.0, 0.5, 0.0)),
    "long_horizon_T100": (96, 100, 40, 2, "tracking", "circle", 0, False, (2.0, 0.0, np.pi / 2, 0.5, 0.0)),
    "lone_variance_tile": (80, 8, 130, 3, "combined", "lane", 3, False, (0.0, 0.0, 0.0, 0.2, 0.0)),
}


@pytest.mark.parametrize("case", sorted(CASES))
@pytest.mark.parametrize("var_path", [0, 1, 3, 4])
def test_edge_case_parity(case, var_path):
    import paper_2411_03289_b200 as G
    K, T, n, R, kind, track, n_obs, split, x0 = CASES[case]
    X, Y, Kp = _gp_data(n, R, seed=n + 7, split_kernels=split)
    gp_o, gp_d = O.GP(X, Y, Kp), G.GpModel.fit(X, Y, Kp)
    assert gp_d.n_groups() == (2 if split else 1)
    obstacles = _obstacles(n_obs, seed=K)
    td, to = _tasks(G, kind, track, obstacles)
    po = O.Planner(K, T, O.ORC_MODEL_GP, gp_o, R, lam=0.1, sigma_sim=(0.09, 0.25), seed=5, threads=0,
                   p_x=0.95)
    pd = G.Planner(G.MppiConfig(samples=K, horizon=T, seed=5), G.GpEnsemble(gp_d, R), p_x=0.95)
    pd.set_variance_path(var_path)
    if R > 1:
        w = np.linspace(1.0, 2.0, R)
        w /= w.sum()
        po.set_terrain_weights(w)
        pd.set_terrain_weights(w)
    x = np.array(x0, dtype=np.float64)
    for t in range(3):
        eps = O.sample_perturbations(K, T, (0.09, 0.25), 5, t)
        pd.inject_noise(eps)
        co, _ = po.plan_step(x, to, eps)
        cd = pd.plan_step(x, td)
        label = f"{case} path {var_path} tick {t}"
        assert_tick_parity(po, pd, label=label)
        np.testing.assert_allclose(cd, co, atol=SEQ_ATOL, err_msg=label + ": command")
        # tick 0 tightens along identical nominals; afterwards the nominals differ within
        # SEQ_ATOL, which a 100-step covariance recursion amplifies on small entries
        rt = TIGHT_RTOL if t == 0 or T <= 40 else 1e-5
        cov_o = po.horizon_covariances()
        np.testing.assert_allclose(pd.horizon_covariances(), cov_o, rtol=rt,
                                   atol=rt * max(np.abs(cov_o).max(), 1e-300), err_msg=label + ": cov")
        if kind != "avoidance":
            np.testing.assert_allclose(pd.lane_radii(), po.lane_radii(), rtol=rt, atol=1e-12,
                                       err_msg=label + ": radii")
        if kind != "tracking" and n_obs:
            np.testing.assert_allclose(pd.obstacle_margins(), po.obstacle_margins(), rtol=rt,
                                       atol=1e-12, err_msg=label + ": margins")
        x = x + np.array([0.01, 0.0, 0.002, 0.0, 0.0])


def test_variance_batch_lone_tile_and_tiny_sizes():
    """The tensor-core variance on 1, 127, 129 and 385 queries (partial and lone tiles)."""
    import paper_2411_03289_b200 as G
    X, Y, Kp = _gp_data(100, 1, seed=3)
    m = G.GpModel.fit(X, Y, Kp)
    rng = np.random.default_rng(1)
    for S in (1, 127, 129, 385):
        q = np.column_stack([rng.uniform(-0.5, 2, S), rng.uniform(-2, 2, S),
                             rng.uniform(-0.5, 2, S), rng.uniform(-2, 2, S)])
        q32 = q.astype(np.float32).astype(np.float64)
        _, v64 = m.predict_batch(q32)
        v = m.variance_batch(q32, 1)[:, 0]
        assert np.abs(v - v64[:, 0]).max() <= 4e-7, S
