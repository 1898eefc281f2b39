"""Batched planner (BASELINE config 4: B independent robots sharing one GP model).

Robot b of a BatchPlanner must behave like a single Planner whose seed is the
robot's seed: flags are bit-identical; per-sample costs agree within the oracle
parity tolerance (the rollout's lane-group layout is sized by the total work, so
the GP-mean partial sums may be grouped differently, and from the second tick on
the nominal sequences differ in the last bits); the softmax sums are taken over a
different block partition, so the command / nominal sequence agree to 1e-12 (first
tick) and 1e-9 afterwards. One robot is also checked against the FP64 CPU oracle with the
device's Philox noise injected (tolerances in tests/helpers.py).
"""
import dataclasses

import numpy as np
import pytest

from oracle import oracle as O
from paper_2411_03289_b200 import workloads as W
from tests.helpers import COST_ATOL, COST_RTOL, SEQ_ATOL, TIGHT_RTOL, assert_tick_parity, oracle_task

pytestmark = pytest.mark.gpu

SUM_TOL = 1e-12


def _robot_tasks(G):
    lane = G.Track.polyline_track([[0.0, 0.0], [60.0, 0.0]], 0.4, False)
    circle = G.Track.circle_track((0.0, 0.0), 2.0, 0.4)
    obs10 = W.random_obstacle_field(10, seed=3)
    obs3 = W.random_obstacle_field(3, seed=5)
    tasks = [G.TrackingTask(circle, 2.0),
             G.AvoidanceTask(obs10, G.GoalSpec((8.0, 0.0), 0.5)),
             G.CombinedTask(lane, 2.0, obs10),
             G.CombinedTask(lane, 1.5, obs3)]
    x0 = np.array([[2.0, 0.0, np.pi / 2, 0.0, 0.0],
                   [0.0, 0.0, 0.0, 0.2, 0.0],
                   [0.0, 0.0, 0.0, 0.0, 0.0],
                   [0.5, 0.1, 0.05, 0.5, 0.1]])
    weights = [[1 / 3, 1 / 3, 1 / 3], [0.6, 0.3, 0.1], [0.2, 0.2, 0.6], [0.0, 1.0, 0.0]]
    return tasks, x0, weights, (obs10, obs3)


def _setup(K=512, T=20, n=256, var_path=None):
    import paper_2411_03289_b200 as G
    X, Y, Kp = W.gp_training_set(n, 3, seed=2)
    gp = G.GpModel.fit(X, Y, Kp)
    tasks, x0, weights, obs = _robot_tasks(G)
    B = len(tasks)
    cfg = G.MppiConfig(samples=K, horizon=T, seed=100)
    bp = G.BatchPlanner(cfg, G.GpEnsemble(gp, 3), B, p_x=0.95)
    singles = []
    for b in range(B):
        p = G.Planner(G.MppiConfig(samples=K, horizon=T, seed=100 + b), G.GpEnsemble(gp, 3), p_x=0.95)
        p.set_terrain_weights(weights[b])
        bp.set_robot_terrain_weights(b, weights[b])
        if var_path is not None:
            p.set_variance_path(var_path)
        singles.append(p)
    if var_path is not None:
        bp.set_variance_path(var_path)
    return G, gp, (X, Y, Kp), bp, singles, tasks, x0, weights, obs


@pytest.mark.parametrize("var_path", [0, 1, 3, 4])
def test_batch_matches_independent_planners(var_path):
    G, gp, _, bp, singles, tasks, x0, weights, _ = _setup(var_path=var_path)
    B = bp.B
    assert bp.robots() == B
    np.testing.assert_array_equal(bp.terrain_weights(), np.array(weights))
    x = x0.copy()
    for t in range(3):
        diags = [G.StepDiagnostics() for _ in range(B)]
        cb = bp.plan_step(x, tasks, diags)
        cs = np.array([singles[b].plan_step(x[b], tasks[b]) for b in range(B)])
        label = f"tick {t}"
        costs = bp.sample_costs()
        flags = bp.flags()
        for b in range(B):
            np.testing.assert_allclose(costs[b], singles[b].sample_costs(), rtol=COST_RTOL, atol=COST_ATOL,
                                       err_msg=f"{label} robot {b} costs")
            fs = singles[b].flags()
            for k in ("viol", "coll", "terminal", "alive"):
                np.testing.assert_array_equal(flags[k][b], fs[k], err_msg=f"{label} robot {b} {k}")
        tol = SUM_TOL if t == 0 else 1e-9
        np.testing.assert_allclose(cb, cs, rtol=tol, atol=tol, err_msg=label + " commands")
        np.testing.assert_allclose(bp.nominal_sequence(), np.array([s.nominal_sequence() for s in singles]),
                                   rtol=tol, atol=tol)
        np.testing.assert_allclose(bp.sample_weights(), np.array([s.sample_weights() for s in singles]),
                                   rtol=1e-7, atol=1e-15)  # exp(-c/lambda) amplifies cost bits by 1/lambda
        # tightening: per-robot blocks run the same arithmetic as the single planner
        # (the nominal sequences feeding it agree to SUM_TOL)
        cov_s = np.array([s.horizon_covariances() for s in singles])  # atol: 1e-9 of the covariance scale
        np.testing.assert_allclose(bp.horizon_covariances(), cov_s, rtol=1e-9, atol=1e-9 * np.abs(cov_s).max())
        rb = bp.lane_radii()
        for b in (0, 2, 3):  # robots with a track
            np.testing.assert_allclose(rb[b], singles[b].lane_radii(), rtol=1e-9, atol=1e-15)
        mb = bp.obstacle_margins()
        assert mb.shape == (B, bp.T, 10)
        for b in (1, 2, 3):
            ms = singles[b].obstacle_margins()
            np.testing.assert_allclose(mb[b, :, : ms.shape[1]], ms, rtol=1e-9, atol=1e-15)
            assert not mb[b, :, ms.shape[1]:].any()
        for b in range(B):
            assert diags[b].nonfinite_samples == 0 and diags[b].ess > 1.0
        x = x + 0.01 * np.arange(1, B + 1)[:, None]


def test_batch_robot_matches_oracle_with_philox_noise():
    G, gp, (X, Y, Kp), bp, singles, tasks, x0, weights, (obs10, obs3) = _setup(K=384, T=16, n=192)
    b = 2  # combined lane task, 10 obstacles
    gp_o = O.GP(X, Y, Kp)
    po = O.Planner(384, 16, O.ORC_MODEL_GP, gp_o, 3, lam=0.1, sigma_sim=(0.09, 0.25), seed=102,
                   threads=0, p_x=0.95)
    po.set_terrain_weights(weights[b])
    w = dataclasses.replace(W.CONFIGS["config2"], task="combined", track="lane")
    to = oracle_task(w, obs10)

    class RobotView:  # the single-planner parity surface of robot b
        def sample_costs(self):
            return bp.sample_costs()[b]

        def flags(self):
            return {k: v[b] for k, v in bp.flags().items()}

        def sample_weights(self):
            return bp.sample_weights()[b]

        def nominal_sequence(self):
            return bp.nominal_sequence()[b]

    x = x0.copy()
    for t in range(2):
        eps = bp.philox_noise(t)
        assert eps.shape == (bp.B, 384, 16, 2)
        co, _ = po.plan_step(x[b], to, eps[b])
        cb = bp.plan_step(x, tasks)
        assert_tick_parity(po, RobotView(), label=f"robot {b} tick {t}")
        np.testing.assert_allclose(cb[b], co, atol=SEQ_ATOL)
        np.testing.assert_allclose(bp.lane_radii()[b], po.lane_radii(), rtol=TIGHT_RTOL, atol=1e-12)
        np.testing.assert_allclose(bp.obstacle_margins()[b], po.obstacle_margins(), rtol=TIGHT_RTOL,
                                   atol=1e-12)


def test_batch_injected_noise_and_errors():
    G, gp, _, bp, singles, tasks, x0, weights, _ = _setup(K=256, T=12, n=128)
    rng = np.random.default_rng(0)
    eps = rng.normal(size=(bp.B, 256, 12, 2)) * np.array([0.3, 0.5])
    bp.inject_noise(eps)
    for b in range(bp.B):
        singles[b].inject_noise(eps[b])
    cb = bp.plan_step(x0, tasks)
    for b in range(bp.B):
        cs = singles[b].plan_step(x0[b], tasks[b])
        np.testing.assert_allclose(bp.sample_costs()[b], singles[b].sample_costs(), rtol=COST_RTOL, atol=COST_ATOL)
        np.testing.assert_allclose(cb[b], cs, rtol=SUM_TOL, atol=SUM_TOL)
    with pytest.raises(ValueError):
        bp.plan_step(x0, tasks[:2])
    with pytest.raises(ValueError):
        bp.set_robot_terrain_weights(bp.B, weights[0])
    bad = x0.copy()
    bad[3, 1] = np.inf
    with pytest.raises(ValueError):
        bp.plan_step(bad, tasks)
    with pytest.raises(ValueError):  # single-robot entry point on a batched handle
        G.Planner.plan_step(bp, x0[0], tasks[0])
    with pytest.raises(ValueError):
        bp.set_shard(0, 10)
