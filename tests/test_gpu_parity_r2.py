"""Parity cases added in round 2 (device through the C ABI vs the FP64 oracle):

- samples that die at different steps of the horizon with live neighbours
  (mppi.cpp:332-346 freeze, :376-377 NaN cost), on the GP rollout and on a GP-free model;
- BASELINE config 4 at its full shape (256 robots x K=4096, T=40, n=512), robots 0 and
  255 against the oracle with their Philox noise;
- BASELINE config 5 at K=65536 against the oracle;
- a signal variance near 1 (the variance error scales with sf2, tests/helpers.py);
- five terrains (10 GP outputs in one kernel group, harness.cpp:242-244);
- command-first mode and re-sharding a planner that has already ticked.
Tolerances: tests/helpers.py.
"""
import dataclasses

import numpy as np
import pytest

from oracle import oracle as O
from paper_2411_03289_b200 import workloads as W
from tests.helpers import (SEQ_ATOL, TIGHT_RTOL, assert_diag_parity, assert_tick_parity, build_pair,
                           cost_atol, oracle_task)

pytestmark = pytest.mark.gpu


def _check_tick(po, pd, to, td, x, eps, label, cost_tol=None):
    """One tick on both sides. A cost tolerance above the default scales the sequence
    tolerance with it (the update is linear in the weights, whose error is |Δc|/λ)."""
    import paper_2411_03289_b200 as G
    from tests.helpers import COST_ATOL
    seq_tol = SEQ_ATOL * max(1.0, (cost_tol or COST_ATOL) / COST_ATOL)
    co, do_ = po.plan_step(x, to, eps)
    dd = G.StepDiagnostics()
    cd = pd.plan_step(x, td, dd)
    assert_tick_parity(po, pd, label=label, cost_tol=cost_tol, seq_tol=seq_tol)
    assert_diag_parity(do_, dd, label=label, **({"cost_tol": cost_tol} if cost_tol else {}))
    np.testing.assert_allclose(cd, co, atol=seq_tol, err_msg=label + ": command")
    return co, do_, cd, dd


def test_mid_horizon_deaths_gp_rollout():
    """Chosen samples get a NaN perturbation at chosen steps k (1..T-1): the clamped control
    is NaN (std::clamp passes NaN), the next state is non-finite, the sample freezes and its
    cost is NaN; the GP queries after the death still run (frozen state, later controls).
    The weighted noise sum multiplies the dead samples' NaN noise by a zero weight exactly
    as update_controls does, so those steps of the sequence become NaN on both sides."""
    w = dataclasses.replace(W.CONFIGS["config2"], name="deaths")
    po, pd, to, td, _ = build_pair(w, samples=512)
    K, T = 512, w.horizon
    eps = O.sample_perturbations(K, T, w.sigma_sim, w.seed, 0)
    rng = np.random.default_rng(7)
    dead = rng.choice(K, size=40, replace=False)
    steps = 1 + rng.integers(0, T - 1, size=40)
    for s, k in zip(dead, steps):
        eps[s, k, int(s) % 2] = np.nan
    pd.inject_noise(eps)
    x = np.array(w.x0)
    co, do_, cd, dd = _check_tick(po, pd, to, td, x, eps, "GP deaths")
    alive = pd.flags()["alive"]
    assert not alive[dead].any() and alive.sum() == K - 40
    assert dd.nonfinite_samples == 40
    assert np.all(np.isfinite(cd))  # no death at k = 0: the command stays finite
    seq = pd.nominal_sequence()
    bad = sorted({int(k) - 1 for k in steps})  # update NaN at k, shifted one step
    assert np.isnan(seq[bad]).any(axis=1).all()


def test_death_at_step_zero_poisons_the_command():
    w = dataclasses.replace(W.CONFIGS["config2"], name="deaths0")
    po, pd, to, td, _ = build_pair(w, samples=256)
    eps = O.sample_perturbations(256, w.horizon, w.sigma_sim, w.seed, 0)
    eps[17, 0, 0] = np.nan
    pd.inject_noise(eps)
    co, do_, cd, dd = _check_tick(po, pd, to, td, np.array(w.x0), eps, "death at k=0")
    assert np.isnan(co[0]) and np.isnan(cd[0]) and dd.nonfinite_samples == 1


def test_overflow_deaths_at_different_steps():
    """Nominal dynamic model from x0 near DBL_MAX with a huge speed state: the position
    overflows after a number of steps that depends on each sample's heading (its own
    omega noise), so samples die at different k with live neighbours (mppi.cpp:362-374).
    The gap to DBL_MAX is chosen on the oracle so that some, not all, samples die."""
    w = dataclasses.replace(W.CONFIGS["config1"], model="nominal", samples=512, horizon=30)
    eps = O.sample_perturbations(512, 30, w.sigma_sim, w.seed, 0)
    to_probe = oracle_task(w, np.zeros((0, 3)))  # kept alive: the C task points into it

    def alive_count(gap):
        po = O.Planner(512, 30, O.ORC_MODEL_NOMINAL, None, 0, lam=w.lam, sigma_sim=w.sigma_sim, seed=w.seed)
        po.plan_step(np.array([1.7976931348623157e308 - gap, 0.0, 1.0, 2.0e306, 0.0]), to_probe, eps)
        return int(po.flags()["alive"].sum())

    lo, hi, x = 1e304, 1e307, None  # bisection: fewer survivors at a smaller gap
    for _ in range(60):
        gap = 0.5 * (lo + hi)
        a = alive_count(gap)
        if 0.1 * 512 < a < 0.9 * 512:
            x = np.array([1.7976931348623157e308 - gap, 0.0, 1.0, 2.0e306, 0.0])
            break
        lo, hi = (gap, hi) if a <= 0.1 * 512 else (lo, gap)
    assert x is not None, "no gap left a mixed alive set"
    po, pd, to, td, _ = build_pair(w)
    pd.inject_noise(eps)
    co, do_, cd, dd = _check_tick(po, pd, to, td, x, eps, "overflow deaths")
    # survivors sit ~1e308 from the track, so their costs overflow to +inf (Eigen norm(),
    # costs.cpp:62-74); the frozen samples' costs are NaN (mppi.cpp:376-377)
    alive = pd.flags()["alive"].astype(bool)
    assert 0 < alive.sum() < 512
    cd_, co_ = pd.sample_costs(), po.costs()
    np.testing.assert_array_equal(np.isnan(cd_), ~alive)
    np.testing.assert_array_equal(np.isnan(co_), ~alive)
    assert np.isposinf(cd_[alive]).all() and np.isposinf(co_[alive]).all()
    assert dd.nonfinite_samples == 512 and np.array_equal(cd, co)


def test_sf2_near_one_parity():
    """Signal variance 0.9: the variance term is ~200x the default workload's; the cost
    tolerance scales with alpha0*T*sf2 (tests/helpers.py)."""
    import paper_2411_03289_b200 as G
    w = dataclasses.replace(W.CONFIGS["config2"], name="sf2")
    X, Y, Kp = W.gp_training_set(256, 3, seed=5)
    Kp[:, 0] = 0.9
    Y = Y * 15.0
    K = 1024
    gp_o, gp_d = O.GP(X, Y, Kp), G.GpModel.fit(X, Y, Kp)
    po = O.Planner(K, w.horizon, O.ORC_MODEL_GP, gp_o, 3, lam=w.lam, sigma_sim=w.sigma_sim, seed=w.seed,
                   p_x=w.p_x)
    pd = G.Planner(G.MppiConfig(samples=K, horizon=w.horizon, lam=w.lam, sigma_sim=w.sigma_sim, seed=w.seed),
                   G.GpEnsemble(gp_d, 3), p_x=w.p_x)
    td, _, obstacles = W.make_task_objects(w, G)
    to = oracle_task(w, obstacles)
    x = np.array(w.x0)
    tol = cost_atol(T=w.horizon, sf2=0.9)
    for t in range(2):
        eps = O.sample_perturbations(K, w.horizon, w.sigma_sim, w.seed, t)
        pd.inject_noise(eps)
        _check_tick(po, pd, to, td, x, eps, f"sf2=0.9 tick {t}", cost_tol=tol)


def test_five_terrains_ten_outputs_one_group():
    """Five terrains share one kernel (harness.cpp:242-244): 10 outputs in a group."""
    import paper_2411_03289_b200 as G
    w = dataclasses.replace(W.CONFIGS["config2"], name="R5", terrains=5, n_points=200)
    po, pd, to, td, data = build_pair(w, samples=512)
    wts = [0.1, 0.3, 0.2, 0.25, 0.15]
    po.set_terrain_weights(wts)
    pd.set_terrain_weights(wts)
    assert data[4].n_groups() == 1 and data[4].n_outputs == 10
    x = np.array(w.x0)
    for t in range(2):
        eps = O.sample_perturbations(512, w.horizon, w.sigma_sim, w.seed, t)
        pd.inject_noise(eps)
        co, _, _, _ = _check_tick(po, pd, to, td, x, eps, f"R=5 tick {t}")
        np.testing.assert_allclose(pd.lane_radii(), po.lane_radii(), rtol=TIGHT_RTOL, atol=1e-12)
    q = data[0][:9] + 0.01
    mo, vo = data[3].predict_batch(q)
    md, vd = data[4].predict_batch(q)
    np.testing.assert_allclose(md, mo, rtol=1e-9, atol=1e-13)


def test_config4_full_shape_robots_0_and_255():
    """BASELINE config 4 at shape: 256 robots x (K=4096, T=40, n=512) in one launch
    sequence; robots 0 and 255 (their own obstacle fields, start offsets and Philox keys)
    against the oracle with the same noise (gpmppi_sample_perturbations with the robot's
    seed = the key the batched planner uses)."""
    import paper_2411_03289_b200 as G
    w = W.CONFIGS["config4"]
    X, Y, Kp = W.gp_training_set(w.n_points, w.terrains, seed=0)
    gp_d, gp_o = G.GpModel.fit(X, Y, Kp), O.GP(X, Y, Kp)
    cfg = G.MppiConfig(samples=w.samples, horizon=w.horizon, lam=w.lam, sigma_sim=w.sigma_sim, seed=w.seed)
    bp = G.BatchPlanner(cfg, G.GpEnsemble(gp_d, w.terrains), w.robots, p_x=w.p_x)
    tasks, x0 = W.make_batch_tasks(w, G)
    cb = bp.plan_step(x0, tasks)
    costs, flags, seq = bp.sample_costs(), bp.flags(), bp.nominal_sequence()
    weights = bp.sample_weights()
    for b in (0, w.robots - 1):
        po = O.Planner(w.samples, w.horizon, O.ORC_MODEL_GP, gp_o, w.terrains, lam=w.lam,
                       sigma_sim=w.sigma_sim, seed=w.seed + b, p_x=w.p_x)
        obstacles = W.random_obstacle_field(w.n_obstacles, seed=3 + b)
        to = oracle_task(w, obstacles)
        eps = G.sample_perturbations(G.MppiConfig(samples=w.samples, horizon=w.horizon, lam=w.lam,
                                                  sigma_sim=w.sigma_sim, seed=w.seed + b), 0)
        co, _ = po.plan_step(x0[b], to, eps)

        class View:
            def sample_costs(self):
                return costs[b]

            def flags(self):
                return {k: v[b] for k, v in flags.items()}

            def sample_weights(self):
                return weights[b]

            def nominal_sequence(self):
                return seq[b]

        assert_tick_parity(po, View(), label=f"config4 robot {b}")
        np.testing.assert_allclose(cb[b], co, atol=SEQ_ATOL)
        np.testing.assert_allclose(bp.lane_radii()[b], po.lane_radii(), rtol=TIGHT_RTOL, atol=1e-12)
        np.testing.assert_allclose(bp.obstacle_margins()[b], po.obstacle_margins(), rtol=TIGHT_RTOL,
                                   atol=1e-12)


def test_config5_k65536_single_tick():
    """BASELINE config 5 at K=65536 (T=40, n=512, combined task) against the oracle."""
    w = W.CONFIGS["config5"]
    po, pd, to, td, _ = build_pair(w)
    eps = pd.philox_noise(0)
    _check_tick(po, pd, to, td, np.array(w.x0), eps, "config5 K=65536")


def test_command_first_mode_matches_synchronous():
    """Command-first returns the same command; the tightening it leaves in flight is
    waited for by the next tick / accessors / wait_tightening (same thresholds)."""
    import paper_2411_03289_b200 as G
    w = W.CONFIGS["config2"]
    _, a, _, td, _ = build_pair(w, samples=1024)
    _, b, _, _, _ = build_pair(w, samples=1024)
    b.set_command_first(True)
    x = np.array(w.x0)
    for t in range(3):
        da, db = G.StepDiagnostics(), G.StepDiagnostics()
        ca = a.plan_step(x, td, da)
        cb = b.plan_step(x, td, db)
        assert np.array_equal(ca, cb)
        if t == 1:
            b.wait_tightening(db)
            assert db.tightening_infeasible == da.tightening_infeasible
            assert db.plan_ms >= db.command_ms
        np.testing.assert_array_equal(a.lane_radii(), b.lane_radii())
        np.testing.assert_array_equal(a.obstacle_margins(), b.obstacle_margins())
        np.testing.assert_array_equal(a.nominal_sequence(), b.nominal_sequence())
        x = x + 0.01


def test_reshard_after_ticks_uses_fresh_buffers():
    """set_shard on a planner that has ticked drops the captured tick graph and frees the
    old per-sample buffers: re-sharding to the full range reproduces a fresh planner."""
    w = W.CONFIGS["config2"]
    _, a, _, td, _ = build_pair(w, samples=768)
    _, b, _, _, _ = build_pair(w, samples=768)
    x = np.array(w.x0)
    a.plan_step(x, td)
    b.plan_step(x, td)
    a.set_shard(0, 768)
    ca, cb = a.plan_step(x, td), b.plan_step(x, td)
    np.testing.assert_array_equal(ca, cb)
    np.testing.assert_array_equal(a.sample_costs(), b.sample_costs())
    eps = a.philox_noise(5)
    a.set_shard(0, 768)
    a.inject_noise(eps)
    b.inject_noise(eps)
    np.testing.assert_array_equal(a.plan_step(x, td), b.plan_step(x, td))
