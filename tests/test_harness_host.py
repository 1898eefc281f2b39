"""Host side of the closed-loop drivers (harness.py): RNG, truth simulator, terrain estimator.

The RNG is pinned bit-exactly to the reference's own rng.hpp through the committed golden
vectors (tests/golden/ref_rng.npz); the estimator cases restate test_terrain.cpp:50-190;
the dynamics are compared with the FP64 oracle. CPU only.
"""
import math
import os

import numpy as np
import pytest

from paper_2411_03289_b200 import gpmppi as G
from paper_2411_03289_b200 import harness as H

GOLD = os.path.join(os.path.dirname(__file__), "golden", "ref_rng.npz")


def test_mt19937_64_standard_known_answer():
    r = H.RngStream(5489)  # [rand.predef]: the 10000th output of default-seeded mt19937_64
    for _ in range(9999):
        r.next_u64()
    assert r.next_u64() == 9981545732273789042


def test_rng_stream_matches_reference_header_bit_exact():
    g = np.load(GOLD)
    for (a, b, c), d in zip(g["triples"], g["derived"]):
        assert H.derive_seed(int(a), int(b), int(c)) == int(d)
    for i, seed in enumerate((0, 5489, 2**64 - 1)):
        r = H.RngStream(seed)
        np.testing.assert_array_equal([r.uniform01() for _ in range(700)], g["uniform"][i])
        r = H.RngStream(seed)
        np.testing.assert_array_equal([r.gaussian() for _ in range(701)], g["gaussian"][i])


def test_step_nominal_matches_oracle(orc):
    rng = np.random.default_rng(3)
    nom = G.NominalParams()
    for _ in range(200):
        s = np.array([rng.uniform(-3, 3), rng.uniform(-3, 3), rng.uniform(-3, 3),
                      rng.uniform(-0.5, 2), rng.choice([0.0, 1e-8, rng.uniform(-2, 2)])])
        u = np.array([rng.uniform(-0.5, 2), rng.uniform(-2, 2)])
        out = np.empty(5)
        orc.lib().orc_step_nominal(orc._ptr(s), orc._ptr(u), orc.Nominal(0.5, 0.35, 0.05),
                                   orc._ptr(out))
        np.testing.assert_array_equal(H.step_nominal(tuple(s), tuple(u), nom), out)


def test_wrap_angle_boundary():  # test_core.cpp:12-19
    assert H.wrap_angle(-math.pi) == math.pi
    assert H.wrap_angle(math.pi) == math.pi
    with pytest.raises(ValueError):
        H.wrap_angle(float("nan"))


def test_true_terrain_step_draws_one_pair_and_follows_lags():
    ter = H.TerrainProfile("x", 0.9, 0.8, 0.5, 0.4, 0.2, 0.0, 0.0)
    r = H.RngStream(1)
    s = H.step_true_terrain((0.0, 0.0, 0.0, 1.0, 0.5), (1.5, 1.0), ter, r, 0.05)
    assert s[3] == 1.0 + 0.1 * (0.9 * 1.5 - 1.0)
    assert s[4] == 0.5 + (0.05 / 0.4) * (0.8 * 1.0 / 1.2 - 0.5)
    r2 = H.RngStream(1)
    r2.gaussian_pair()
    assert r.next_u64() == r2.next_u64()  # exactly two uniforms consumed


# ---------------------------------------------------------------- terrain.cpp
def _random_buffer(rng, rows, m):  # test_terrain.cpp:33-44
    buf = H.HistoryBuffer(max(rows, 1), m)
    for _ in range(rows):
        pred = np.empty((m, 2))
        for i in range(m):
            pred[i, 0] = rng.uniform(-1, 1)
            pred[i, 1] = rng.uniform(-1, 1)
        meas = (rng.uniform(-1, 1), rng.uniform(-1, 1))
        buf.push(meas, pred)
    return buf


def _objective(buf, w, prev, gamma):
    return (np.sum((buf.y_v() - buf.f_v() @ w) ** 2) + np.sum((buf.y_omega() - buf.f_omega() @ w) ** 2)
            + gamma * np.abs(w - prev).sum())


def _grid_oracle(buf, prev, gamma, res):  # test_terrain.cpp:18-31
    best = math.inf
    for w0 in np.arange(0.0, 1.0 + 1e-12, res):
        for w1 in np.arange(0.0, 1.0 - w0 + 1e-12, res):
            w = np.array([w0, w1, max(1.0 - w0 - w1, 0.0)])
            best = min(best, _objective(buf, w, prev, gamma))
    return best


def test_history_buffer_fifo():  # test_terrain.cpp:50-68
    buf = H.HistoryBuffer(3, 2)
    assert buf.size() == 0
    for i in range(3):
        buf.push((float(i), float(-i)), np.full((2, 2), float(i)))
    assert buf.size() == 3 and buf.y_v()[0] == 0.0
    buf.push((3.0, -3.0), np.full((2, 2), 99.0))
    assert buf.size() == 3
    assert buf.y_v()[0] == 1.0 and buf.y_v()[2] == 3.0
    assert buf.f_v()[2, 0] == 99.0 and buf.f_omega()[2, 1] == 99.0
    with pytest.raises(ValueError):
        buf.push((0.0, 0.0), np.zeros((3, 2)))


def test_project_simplex_worked_examples():  # test_terrain.cpp:70-79
    z = np.array([0.2, 0.3, 0.5])
    assert np.linalg.norm(H.project_simplex(z) - z) <= 1e-15
    assert np.linalg.norm(H.project_simplex([2.0, 0.0, 0.0]) - [1, 0, 0]) <= 1e-15
    assert np.linalg.norm(H.project_simplex([0.5, 0.5, 0.5]) - 1.0 / 3) <= 1e-12
    with pytest.raises(ValueError):
        H.project_simplex([np.nan, 1.0])


def test_project_simplex_is_a_projection():  # test_terrain.cpp:81-98
    rng = H.RngStream(3)
    for _ in range(300):
        z = np.array([rng.uniform(-3, 3) for _ in range(4)])
        p = H.project_simplex(z)
        assert p.min() >= 0.0 and abs(p.sum() - 1.0) <= 1e-12
        assert np.linalg.norm(H.project_simplex(p) - p) <= 1e-12
        for _ in range(5):
            q = np.array([rng.uniform(0, 1) for _ in range(4)])
            q /= q.sum()
            assert np.sum((z - p) ** 2) <= np.sum((z - q) ** 2) + 1e-9


def test_solve_weights_identifies_generating_terrain():  # test_terrain.cpp:100-118
    m, rows = 3, 20
    buf = H.HistoryBuffer(rows, m)
    for r in range(rows):
        pred = np.array([[math.sin(0.3 * r + i), math.cos(0.2 * r - i)] for i in range(m)])
        buf.push((pred[1, 0], pred[1, 1]), pred)
    res = H.solve_weights(buf, np.full(m, 1.0 / m), H.WeightSolverConfig(gamma=0.0))
    assert H.on_simplex(res.weights, 1e-9) and res.weights[1] >= 0.99


def test_identical_columns_keep_prev():  # test_terrain.cpp:120-135
    buf = H.HistoryBuffer(8, 3)
    for _ in range(8):
        buf.push((0.6, -0.1), np.column_stack([np.full(3, 0.5), np.full(3, -0.2)]))
    prev = np.array([0.2, 0.5, 0.3])
    res = H.solve_weights(buf, prev, H.WeightSolverConfig(gamma=0.1))
    assert np.abs(res.weights - prev).max() <= 1e-9


def test_huge_gamma_pins_prev():  # test_terrain.cpp:137-146
    buf = _random_buffer(H.RngStream(7), 12, 3)
    prev = np.array([0.7, 0.2, 0.1])
    res = H.solve_weights(buf, prev, H.WeightSolverConfig(gamma=1e9))
    assert np.abs(res.weights - prev).max() <= 1e-9


def test_empty_buffer_returns_prev_flagged():  # test_terrain.cpp:148-154
    prev = np.full(3, 1.0 / 3)
    res = H.solve_weights(H.HistoryBuffer(5, 3), prev, H.WeightSolverConfig())
    assert res.buffer_empty and np.array_equal(res.weights, prev)
    with pytest.raises(ValueError):
        H.solve_weights(H.HistoryBuffer(5, 3), np.array([0.5, 0.6, 0.0]), H.WeightSolverConfig())


def test_solver_matches_exhaustive_grid():  # test_terrain.cpp:156-170
    rng = H.RngStream(11)
    for trial in range(25):
        buf = _random_buffer(rng, 5 + trial % 15, 3)
        prev = H.project_simplex([rng.uniform(0, 1) for _ in range(3)])
        gamma = 0.0 if trial % 2 == 0 else 0.1
        res = H.solve_weights(buf, prev, H.WeightSolverConfig(gamma=gamma))
        assert res.objective <= _grid_oracle(buf, prev, gamma, 0.005) + 1e-6
        assert H.on_simplex(res.weights, 1e-9)


def test_solver_row_permutation_invariant():  # test_terrain.cpp:172-190
    rng = H.RngStream(13)
    m, rows = 3, 10
    preds, meas = [], []
    for _ in range(rows):
        preds.append(np.array([[rng.uniform(-1, 1), rng.uniform(-1, 1)] for _ in range(m)]))
        meas.append((rng.uniform(-1, 1), rng.uniform(-1, 1)))
    fwd, rev = H.HistoryBuffer(rows, m), H.HistoryBuffer(rows, m)
    for r in range(rows):
        fwd.push(meas[r], preds[r])
    for r in reversed(range(rows)):
        rev.push(meas[r], preds[r])
    prev = np.full(m, 1.0 / m)
    a = H.solve_weights(fwd, prev, H.WeightSolverConfig())
    b = H.solve_weights(rev, prev, H.WeightSolverConfig())
    assert np.abs(a.weights - b.weights).max() <= 1e-9


# ---------------------------------------------------------------- scenarios
def test_random_obstacle_field_respects_clearances():
    goal = G.GoalSpec((8.0, 0.0), 0.5)
    obs = H.random_obstacle_field(H.RngStream(H.derive_seed(4, 3)), 10, goal=goal)
    assert len(obs) == 10
    for o in obs:
        assert 1.5 <= o.center[0] <= 6.5 and -2.5 <= o.center[1] <= 2.5
        assert 0.25 <= o.radius <= 0.5
        assert math.hypot(*o.center) >= o.radius + 0.5
        assert math.hypot(o.center[0] - 8.0, o.center[1]) >= o.radius + 1.0


def test_make_scenario_canonical_starts(orc):
    sc = H.make_scenario("tracking", "circle")
    assert sc.start == (2.0, 0.0, 0.5 * math.pi, 0.0, 0.0)
    assert H.centerline_distance(sc.track, (3.0, 0.0)) == 1.0
    sq = H.make_scenario("tracking", "square")
    assert sq.start[:3] == (0.0, -3.125, 0.0)
    assert H.centerline_distance(sq.track, (0.0, 0.0)) == 3.125
    av = H.make_scenario("avoidance", seed=9)
    assert av.start == (0.0, 0.0, 0.0, 0.0, 0.0) and len(av.obstacles) == 5
    assert H.make_scenario("avoidance", seed=9).obstacles == av.obstacles  # (config, seed) pins it
    sch = H.Scenario(schedule=[(0.0, 0), (5.0, 2)])
    assert sch.terrain_at(4.99) == 0 and sch.terrain_at(5.0) == 2


def test_latency_summary_and_rmse():
    s = H.summarize_latency([3.0, 1.0, 2.0, 4.0])
    assert (s.mean_ms, s.median_ms, s.max_ms) == (2.5, 2.5, 4.0)
    tr = G.Track.circle_track((0.0, 0.0), 2.0, 0.4)
    assert H.compute_rmse([(2.0, 0.0), (0.0, 3.0)], tr) == math.sqrt(0.5)
    with pytest.raises(ValueError):
        H.compute_rmse([], tr)


def test_training_data_residuals_and_kernel_grid():
    nom = G.NominalParams()
    ter = H.default_terrains()[2]
    X, R = H.generate_training_data(ter, nom, G.ControlBounds(), 60, H.RngStream(1))
    assert X.shape == (60, 4) and R.shape == (60, 2)
    assert np.abs(R).max() < 0.5 and np.abs(R).max() > 0.0
    from oracle import oracle as O  # the CPU restatement (the device grid: test_gpu_kernel_grid.py)
    sv, ls, nv, lml = O.select_kernel_grid(X, R)
    assert sv > 0 and nv > 0 and min(ls) > 0 and np.isfinite(lml)
