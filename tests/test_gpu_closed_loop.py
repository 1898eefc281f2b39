"""Closed-loop drivers on the B200 planner (harness.cpp:298-421; acceptance.cpp:335-420 shape).

Every tick plans on the device, steps the true-terrain simulator and re-solves the terrain
weights. Runs are shortened (distance budget / trial count) so the test takes seconds; the
acceptance criteria's orderings are checked where a short run supports them.
"""
import math

import numpy as np
import pytest

from paper_2411_03289_b200 import gpmppi as G
from paper_2411_03289_b200 import harness as H

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def trained():
    cfg = H.ExperimentConfig(n_points=200)
    return cfg, H.train_models(cfg, seed=0)


def test_tracking_closed_loop_gp_beats_unicycle_on_grass(trained):
    cfg, models = trained
    out = {}
    for kind in ("gp", "unicycle"):
        c = H.ExperimentConfig(**{**cfg.__dict__, "planner": kind})
        sc = H.make_scenario("tracking", "circle", schedule=[(0.0, 2)], distance_budget=15.0,
                             max_duration=40.0)
        trace = []
        m = H.run_tracking_experiment(c, sc, models, seed=7, trace=trace)
        assert not m.aborted, m.abort_reason
        assert m.success and m.ticks == len(trace)
        assert m.latency.median_ms > 0.0 and m.latency.max_ms >= m.latency.median_ms
        out[kind] = m
        if kind == "gp":  # estimator lands on the simplex and moves toward grass
            w = np.array([r.terrain_weights for r in trace])
            assert np.allclose(w.sum(1), 1.0, atol=1e-12) and w.min() >= 0.0
            assert w[-1, 2] > 1.0 / 3
    assert out["gp"].rmse < out["unicycle"].rmse  # acceptance.cpp:362 ordering


def test_avoidance_closed_loop_reaches_goal(trained):
    cfg, models = trained
    sc = H.make_scenario("avoidance", seed=3, schedule=[(0.0, 1)], max_duration=30.0)
    m = H.run_avoidance_experiment(cfg, sc, models, seed=3)
    assert not m.aborted, m.abort_reason
    assert m.time_to_goal > 0.0 and math.isfinite(m.min_obstacle_clearance)
    assert m.success == (m.collision_count == 0)


def test_per_terrain_prediction_is_nominal_plus_residual():  # test_terrain.cpp:192-210
    rng = H.RngStream(17)
    x = np.array([[rng.uniform(-0.5, 2), rng.uniform(-2, 2), rng.uniform(-0.5, 2), rng.uniform(-2, 2)]
                  for _ in range(40)])
    model = G.GpModel.fit(x, np.zeros((40, 4)), [G.KernelParams(noise_var=1e-6)] * 4)
    pred = H.per_terrain_mean_prediction(model, (1.0, 0.5, 1.5, -0.5), G.NominalParams(0.5, 0.35, 0.05))
    assert pred.shape == (2, 2)
    np.testing.assert_allclose(pred[:, 0], 1.0 + 0.1 * 0.5, rtol=1e-9)
    np.testing.assert_allclose(pred[:, 1], 0.5 + (0.05 / 0.35) * (-1.0), rtol=1e-9)


def test_kind_mismatch_raises(trained):
    cfg, models = trained
    with pytest.raises(ValueError):
        H.run_tracking_experiment(cfg, H.make_scenario("avoidance"), models, 0)
    with pytest.raises(ValueError):
        H.run_avoidance_experiment(cfg, H.make_scenario("tracking"), models, 0)


def test_python_entry_points_match_reference_bindings():  # module.cpp:183-210, test_smoke.py
    m = H.run_tracking(seed=1, planner="unicycle", distance_budget=5.0)
    assert set(m) >= {"rmse", "success", "ticks", "latency_median_ms", "abort_reason"}
    assert m["success"] and not m["aborted"]
    a = H.run_avoidance(seed=2, planner="gp", max_duration=20.0)
    assert a["ticks"] > 0 and not a["aborted"]
    with pytest.raises(RuntimeError, match="cannot open"):  # std::runtime_error, config.cpp:189-191
        H.run_tracking(config_path="no-such-cfg.json")
