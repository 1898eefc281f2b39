"""Device (sm_100a, through the C ABI) vs FP64 CPU oracle on identical inputs.

Noise: the reference's own mt19937_64 tensors (oracle restatement, pinned to
the reference header) are injected into the device planner; the Philox mode is
checked by materialising the device noise and injecting it into the oracle.
Tolerances are stated in tests/helpers.py.
"""
import dataclasses

import numpy as np
import pytest

from oracle import oracle as O
from paper_2411_03289_b200 import workloads as W
from tests.helpers import (COST_ATOL, SEQ_ATOL, TIGHT_RTOL, assert_diag_parity, assert_tick_parity,
                           build_pair)

pytestmark = pytest.mark.gpu


def _run_ticks(w, ticks=3, samples=None, philox=False, gp_seed=0, flags_exact=True, var_path=None):
    import paper_2411_03289_b200 as G
    po, pd, to, td, _ = build_pair(w, gp_seed=gp_seed, samples=samples, var_path=var_path)
    K, T = po.K, po.T
    x = np.array(w.x0, dtype=np.float64)
    for t in range(ticks):
        if philox:
            eps = pd.philox_noise(t)
        else:
            eps = O.sample_perturbations(K, T, w.sigma_sim, w.seed, t)
            pd.inject_noise(eps)
        co, do_ = po.plan_step(x, to, eps)
        dd = G.StepDiagnostics()
        cd = pd.plan_step(x, td, dd)
        label = f"{w.name} tick {t}"
        assert_tick_parity(po, pd, flags_exact=flags_exact, label=label)
        assert_diag_parity(do_, dd, label=label)
        np.testing.assert_allclose(cd, co, atol=SEQ_ATOL, err_msg=label + ": command")
        if w.task != "avoidance":
            np.testing.assert_allclose(pd.lane_radii(), po.lane_radii(), rtol=TIGHT_RTOL,
                                       atol=1e-12, err_msg=label + ": lane radii")
        if w.task != "tracking" and w.n_obstacles:
            np.testing.assert_allclose(pd.obstacle_margins(), po.obstacle_margins(),
                                       rtol=TIGHT_RTOL, atol=1e-12, err_msg=label + ": margins")
        cov_o = po.horizon_covariances()
        np.testing.assert_allclose(pd.horizon_covariances(), cov_o, rtol=TIGHT_RTOL,
                                   atol=TIGHT_RTOL * np.abs(cov_o).max(),
                                   err_msg=label + ": covariances")
        x = _advance(x, co)
    return po, pd


def _advance(x, u):
    out = np.empty(5)
    O.lib().orc_step_nominal(O._ptr(np.asarray(x, dtype=np.float64)),
                             O._ptr(np.asarray(u, dtype=np.float64)), O.Nominal(0.5, 0.35, 0.05),
                             O._ptr(out))
    return out


def test_gp_predict_matches_oracle():
    import paper_2411_03289_b200 as G
    X, Y, Kp = W.gp_training_set(96, 3, seed=4)
    go, gd = O.GP(X, Y, Kp), G.GpModel.fit(X, Y, Kp)
    rng = np.random.default_rng(1)
    q = np.column_stack([rng.uniform(-0.5, 2, 200), rng.uniform(-2, 2, 200),
                         rng.uniform(-0.5, 2, 200), rng.uniform(-2, 2, 200)])
    mo, vo = go.predict_batch(q)
    md, vd = gd.predict_batch(q)
    np.testing.assert_allclose(md, mo, rtol=1e-9, atol=1e-13)
    np.testing.assert_allclose(vd, vo, rtol=1e-7, atol=1e-13)
    assert gd.n_groups() == 1 and gd.n_points == 96 and gd.n_outputs == 6
    for o in range(6):
        assert gd.log_marginal_likelihood(o) == pytest.approx(go.lml(o), rel=1e-10)


def test_gp_predict_two_groups_and_closed_form():  # test_gp.cpp:65-78,157-183
    import paper_2411_03289_b200 as G
    m = G.GpModel.fit(np.zeros((1, 4)), np.array([[2.0]]), [G.KernelParams(1.0, (1, 1, 1, 1), 1.0)])
    mean, var = m.predict(np.zeros(4))
    assert mean[0] == pytest.approx(1.0, rel=1e-12) and var[0] == pytest.approx(0.5, rel=1e-12)
    rng = np.random.default_rng(13)
    x = np.column_stack([rng.uniform(-0.5, 2, 100), rng.uniform(-2, 2, 100),
                         rng.uniform(-0.5, 2, 100), rng.uniform(-2, 2, 100)])
    y = np.column_stack([np.sin(x[:, 0]), np.cos(x[:, 1]), 0.2 * x[:, 2]])
    ks = [[0.5, 1, 1, 1, 1, 1e-4]] * 2 + [[0.5, 2, 2, 2, 2, 1e-4]]
    gd, go = G.GpModel.fit(x, y, ks), O.GP(x, y, ks)
    assert gd.n_groups() == 2
    q = x[:17] + 0.05
    np.testing.assert_allclose(gd.predict_batch(q)[0], go.predict_batch(q)[0], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(gd.predict_batch(q)[1], go.predict_batch(q)[1], rtol=1e-6, atol=1e-12)


def test_reference_ragged_chunk_case():
    """test_mppi.cpp:181-229 shape: K=257 (ragged), T=6, n=60, 2 terrains (0.3, 0.7)."""
    import paper_2411_03289_b200 as G
    w = dataclasses.replace(W.CONFIGS["config3"], name="ragged", samples=257, horizon=6,
                            n_points=60, terrains=2, seed=12345)
    po, pd, to, td, _ = build_pair(w, gp_seed=17)
    po.set_terrain_weights([0.3, 0.7])
    pd.set_terrain_weights([0.3, 0.7])
    x0 = np.array([2.0, 0.0, 1.5707963267948966, 1.0, 0.5])
    for t in range(2):
        eps = O.sample_perturbations(257, 6, w.sigma_sim, w.seed, t)
        pd.inject_noise(eps)
        co, _ = po.plan_step(x0, to, eps)
        cd = pd.plan_step(x0, td)
        assert_tick_parity(po, pd, label=f"ragged tick {t}")
        np.testing.assert_allclose(cd, co, atol=SEQ_ATOL)


@pytest.mark.parametrize("task", ["tracking", "avoidance", "combined"])
def test_config2_shape_reduced_K_injected_reference_noise(task):
    w = dataclasses.replace(W.CONFIGS["config2"], task=task, track="lane" if task != "tracking" else "circle",
                            x0=(0.0, 0.0, 0.0, 0.0, 0.0) if task != "tracking" else (2.0, 0.0, np.pi / 2, 0.0, 0.0))
    _run_ticks(w, ticks=3, samples=512)


@pytest.mark.parametrize("var_path", [0, 1, 3, 4])
def test_config2_variance_paths_parity(var_path):
    """FFMA and tcgen05 3xTF32 variance paths both meet the stated cost tolerance."""
    _run_ticks(W.CONFIGS["config2"], ticks=2, samples=2048, var_path=var_path)


@pytest.mark.parametrize("var_path", [1, 3, 4])
def test_config3_shape_parity_tc(var_path):
    """n=2048, T=60 multi-terrain (BASELINE config 3 shape) at reduced K: 3xTF32 and the
    default 3xFP16 variance through plan_step."""
    _run_ticks(W.CONFIGS["config3"], ticks=1, samples=512, var_path=var_path)


def test_config3_default_path_k4096():
    """Config 3 (T=60, n=2048) through plan_step on the default 3xFP16 variance at K=4096."""
    _run_ticks(W.CONFIGS["config3"], ticks=1, samples=4096)


def test_config2_philox_noise_parity():
    _run_ticks(W.CONFIGS["config2"], ticks=2, samples=1024, philox=True)


@pytest.mark.parametrize("model", ["nominal", "unicycle", "edd5"])
def test_gp_free_models(model):
    w = dataclasses.replace(W.CONFIGS["config1"], model=model)
    _run_ticks(w, ticks=3)


def test_full_config2_single_tick_parity():
    """Full headline shape (K=4096, T=40, n=512, 10 obstacles), reference noise."""
    _run_ticks(W.CONFIGS["config2"], ticks=1)


def test_determinism_and_noise_materialisation():
    import paper_2411_03289_b200 as G
    w = W.CONFIGS["config2"]
    _, pd1, _, td, _ = build_pair(w, samples=700)
    _, pd2, _, _, _ = build_pair(w, samples=700)
    x0 = np.array(w.x0)
    c1 = [pd1.plan_step(x0, td) for _ in range(3)]
    c2 = [pd2.plan_step(x0, td) for _ in range(3)]
    assert np.array_equal(np.array(c1), np.array(c2))
    e0 = pd1.philox_noise(0)
    assert e0.shape == (700, 40, 2)
    assert abs(e0[..., 0].mean()) < 4 * 0.3 / np.sqrt(e0[..., 0].size)
    assert e0[..., 0].std() == pytest.approx(0.3, rel=0.02)
    assert e0[..., 1].std() == pytest.approx(0.5, rel=0.02)


def test_all_nonfinite_batch_is_a_zero_update():  # mppi.cpp:130-135, test_mppi.cpp:97-107
    import paper_2411_03289_b200 as G
    w = dataclasses.replace(W.CONFIGS["config1"], model="nominal", samples=300, horizon=5)
    po, pd, to, td, _ = build_pair(w)
    x0 = np.array([1.7976e308, 0.0, 0.0, 1.5e308, 0.0])  # x overflows on the first step
    eps = O.sample_perturbations(300, 5, w.sigma_sim, w.seed, 0)
    pd.inject_noise(eps)
    d = G.StepDiagnostics()
    co, do_ = po.plan_step(x0, to, eps)
    cd = pd.plan_step(x0, td, d)
    assert do_["nonfinite_samples"] == 300 and d.nonfinite_samples == 300
    assert d.ess == 0.0 and d.weight_entropy == 0.0 and np.isinf(d.best_cost)
    np.testing.assert_array_equal(cd, co)
    assert not pd.flags()["alive"].any()


def test_errors_map_to_reference_exceptions():
    import paper_2411_03289_b200 as G
    with pytest.raises(ValueError):
        G.Planner(G.MppiConfig(samples=0), G.UnicycleBaseline())
    with pytest.raises(ValueError):
        G.Planner(G.MppiConfig(samples=8, lam=0.0), G.UnicycleBaseline())
    p = G.Planner(G.MppiConfig(samples=8, horizon=4), G.UnicycleBaseline())
    t = G.TrackingTask(G.Track.circle_track((0, 0), 2.0, 0.4), 1.0)
    with pytest.raises(ValueError):
        p.plan_step([np.nan, 0, 0, 0, 0], t)
    with pytest.raises(ValueError):
        p.plan_step([0, 0, 0, 0, 0], G.TrackingTask(G.Track.circle_track((0, 0), 2.0, -1.0), 1.0))
    try:  # test_gp.cpp:205-220: duplicate rows either fit via jitter or raise naming it
        m = G.GpModel.fit(np.ones((2, 4)), np.ones((2, 1)), [G.KernelParams(1.0, (1, 1, 1, 1), 1e-300)])
        assert 0.0 < m.group_jitter(0) <= 1e-6
    except RuntimeError as e:
        assert "jitter" in str(e)


def test_model_save_load_roundtrip(tmp_path):  # test_gp.cpp:233-256
    import paper_2411_03289_b200 as G
    X, Y, Kp = W.gp_training_set(48, 1, seed=21)
    m = G.GpModel.fit(X, Y, Kp)
    path = str(tmp_path / "model.bin")
    m.save(path)
    b = G.GpModel.load(path)
    Xb, Yb = b.training_data()
    assert np.array_equal(Xb, X) and np.array_equal(Yb, Y)
    q = np.array([[0.3, 0.1, 1.2, -0.4]])
    assert np.array_equal(m.predict_batch(q)[0], b.predict_batch(q)[0])
    assert np.array_equal(m.predict_batch(q)[1], b.predict_batch(q)[1])
