"""Reference free functions (mppi.hpp:60-79) on the device vs the reference's own
known-answer tests (test_mppi.cpp:39-179) and the FP64 oracle.

The device sums in a different order than the reference's sequential loops
(block reductions), so sums agree to 1e-12 relative, not bit-for-bit; the
rollout is FP64 end to end (tolerance 1e-12 vs the oracle, 1e-9 as the
reference test states for the zero-residual case).
"""
import math

import numpy as np
import pytest

from oracle import oracle as O
from paper_2411_03289_b200 import workloads as W

pytestmark = pytest.mark.gpu


def test_trajectory_weights_known_answers():  # test_mppi.cpp:70-117
    import paper_2411_03289_b200 as G
    w = G.trajectory_weights(np.full(8, 3.0), 0.5)
    assert w.sum() == pytest.approx(1.0, rel=1e-12) and np.allclose(w, 0.125, rtol=1e-12)
    w = G.trajectory_weights([0.0, 0.1], 0.1)
    z = 1 + math.exp(-1)
    assert w[0] == pytest.approx(1 / z, rel=1e-12) and w[1] == pytest.approx(math.exp(-1) / z, rel=1e-12)
    assert G.trajectory_weights([5.0, 1.0, 9.0], 1e-6)[1] == pytest.approx(1.0, rel=1e-9)
    a = G.trajectory_weights([1, 2, 3, 4], 0.7)
    b = G.trajectory_weights(np.array([1, 2, 3, 4]) + 1e6, 0.7)
    assert np.abs(a - b).max() <= 1e-12
    w = G.trajectory_weights([1.0, np.inf, np.nan], 0.5)
    assert w[0] == pytest.approx(1.0) and w[1] == 0 and w[2] == 0
    assert np.abs(G.trajectory_weights([np.nan] * 3, 0.5)).max() == 0.0
    with pytest.raises(ValueError):
        G.trajectory_weights([1.0, 2.0], 0.0)
    rng = np.random.default_rng(5)
    for _ in range(10):
        c = rng.uniform(0, 10, 4097)
        c[rng.integers(0, 4097, 20)] = np.nan
        np.testing.assert_allclose(G.trajectory_weights(c, 0.3), O.trajectory_weights(c, 0.3),
                                   rtol=1e-12, atol=1e-300)


def test_update_controls_and_shift_known_answers():  # test_mppi.cpp:119-160
    import paper_2411_03289_b200 as G
    nom = np.array([[1.0, 0.0]] * 3)
    e1 = np.zeros((1, 3, 2))
    e1[0, 1, 0] = 0.3
    assert G.update_controls(nom, e1, [1.0])[1, 0] == pytest.approx(1.3)
    out = G.update_controls(nom, np.full((1, 3, 2), 100.0), [1.0])
    assert out[0, 0] == 2.0 and out[0, 1] == 2.0
    with pytest.raises(ValueError):
        G.update_controls(nom, np.zeros((2, 3, 2)), [1.0])
    seq = np.array([[1, 0], [2, 0], [3, 0]], dtype=float)
    s1 = G.shift_horizon(seq)
    assert s1[0, 0] == 2 and s1[2, 0] == 3
    assert (G.shift_horizon(s1)[:, 0] == 3).all()
    with pytest.raises(ValueError):
        G.shift_horizon(np.zeros((0, 2)))
    rng = np.random.default_rng(3)
    K, T = 2048, 40
    eps = rng.normal(size=(K, T, 2)) * [0.3, 0.5]
    w = O.trajectory_weights(rng.uniform(0, 5, K), 0.1)
    nom = rng.uniform(-0.4, 1.5, (T, 2))
    np.testing.assert_allclose(G.update_controls(nom, eps, w), O.update_controls(nom, eps, w),
                               rtol=1e-13, atol=1e-14)
    np.testing.assert_array_equal(G.shift_horizon(nom), O.shift_horizon(nom))


def test_zero_residual_rollout_equals_nominal():  # test_mppi.cpp:162-179
    import paper_2411_03289_b200 as G
    r = np.random.default_rng(77)
    x = np.column_stack([r.uniform(-0.5, 2, 24), r.uniform(-2, 2, 24), r.uniform(-0.5, 2, 24),
                         r.uniform(-2, 2, 24)])
    gp = G.GpModel.fit(x, np.zeros((24, 6)), [G.KernelParams(1.0, (1, 1, 1, 1), 1e-6)] * 6)
    r9 = np.random.default_rng(9)
    seq = np.column_stack([r9.uniform(0, 2, 10), r9.uniform(-1, 1, 10)])
    x0 = np.array([0.0, 0.0, 0.3, 1.0, 0.2])
    res = G.rollout(x0, seq, G.GpEnsemble(gp, 3))
    s = x0.copy()
    for k in range(10):
        nxt = np.empty(5)
        O.lib().orc_step_nominal(O._ptr(s), O._ptr(np.ascontiguousarray(seq[k])),
                                 O.Nominal(0.5, 0.35, 0.05), O._ptr(nxt))
        s = nxt
        assert abs(res.states[k + 1, 0] - s[0]) <= 1e-9 and abs(res.states[k + 1, 3] - s[3]) <= 1e-9
        assert np.abs(res.corrections[k, :2]).max() <= 1e-9
    with pytest.raises(ValueError):
        G.rollout(x0, seq, G.GpEnsemble(gp, 3), weights=[0.5, 0.5, 0.5])


@pytest.mark.parametrize("model", ["gp", "unicycle", "edd5", "nominal"])
def test_rollout_matches_oracle(model):
    import paper_2411_03289_b200 as G
    r = np.random.default_rng(21)
    seq = np.column_stack([r.uniform(-0.5, 2, 30), r.uniform(-2, 2, 30)])
    x0 = np.array([0.3, -0.2, 0.4, 0.8, -0.1])
    edd = (0.9, 0.95, 0.02, -0.2, 0.21)
    if model == "gp":
        X, Y, Kp = W.gp_training_set(200, 3, seed=5)
        gd, go = G.GpModel.fit(X, Y, Kp), O.GP(X, Y, Kp)
        w = [0.2, 0.5, 0.3]
        res = G.rollout(x0, seq, G.GpEnsemble(gd, 3), weights=w)
        st, corr = O.rollout(x0, seq, O.ORC_MODEL_GP, go, 3, w)
        np.testing.assert_allclose(res.corrections[:, 2:], corr[:, 2:], rtol=1e-7, atol=1e-13)
    else:
        dm = {"unicycle": G.UnicycleBaseline(), "edd5": G.Edd5Baseline(G.Edd5Params(*edd), 0.4),
              "nominal": G.NominalDynamic()}[model]
        kind = {"unicycle": O.ORC_MODEL_UNICYCLE, "edd5": O.ORC_MODEL_EDD5, "nominal": O.ORC_MODEL_NOMINAL}[model]
        res = G.rollout(x0, seq, dm)
        st, corr = O.rollout(x0, seq, kind, edd5=edd, track_width=0.4)
    np.testing.assert_allclose(res.states, st, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(res.corrections[:, :2], corr[:, :2], rtol=1e-10, atol=1e-15)


def test_sample_perturbations_philox():  # test_mppi.cpp:39-68 (determinism + calibration)
    import paper_2411_03289_b200 as G
    cfg = G.MppiConfig(samples=3000, horizon=20, seed=4)
    a, b = G.sample_perturbations(cfg, 7), G.sample_perturbations(cfg, 7)
    assert a.shape == (3000, 20, 2) and np.array_equal(a, b)
    assert not np.array_equal(a, G.sample_perturbations(cfg, 8))
    assert a[..., 0].std() == pytest.approx(0.3, rel=0.02) and a[..., 1].std() == pytest.approx(0.5, rel=0.02)
    p = G.Planner(cfg, G.UnicycleBaseline())
    np.testing.assert_array_equal(p.philox_noise(7), a)  # the planner's own noise stream
