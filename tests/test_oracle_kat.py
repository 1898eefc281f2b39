"""Pins the FP64 CPU oracle against the reference's own known answers.

Every case below restates an inline known-answer test of the reference suite
(cited file:line under /root/reference/proj/tests) or a golden vector produced
by the reference's own RNG header (tests/golden/ref_rng.npz, made by
tests/golden/make_golden.py from oracle/_ref). CPU only.
"""
import math
import os

import numpy as np
import pytest

from oracle import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden", "ref_rng.npz")
NOM = O.Nominal(0.5, 0.35, 0.05)


def f(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def P(a):
    return O._ptr(a)


# ---------------------------------------------------------------- rng.hpp
def test_rng_matches_reference_header_bit_exact():
    g = np.load(GOLD)
    L = O.lib()
    for (a, b, c), d in zip(g["triples"], g["derived"]):
        assert L.orc_derive_seed(int(a), int(b), int(c)) == int(d)
    for i, seed in enumerate((0, 5489, 2**64 - 1)):
        u = np.empty(700)
        gs = np.empty(701)
        L.orc_uniform_stream(seed, 700, P(u))
        L.orc_gaussian_stream(seed, 701, P(gs))
        np.testing.assert_array_equal(u, g["uniform"][i])
        np.testing.assert_array_equal(gs, g["gaussian"][i])
    for j, (K, T, sv2, sw2, seed, tick) in enumerate(g["cases"]):
        K, T, seed, tick = int(K), int(T), int(seed), int(tick)
        eps = O.sample_perturbations(K, T, (sv2, sw2), seed, tick)
        np.testing.assert_array_equal(eps, g[f"eps{j}"])


def test_noise_determinism_and_calibration():  # test_mppi.cpp:39-68
    a = O.sample_perturbations(100, 4, (0.09, 0.25), 12345, 3)
    b = O.sample_perturbations(100, 4, (0.09, 0.25), 12345, 3)
    c = O.sample_perturbations(100, 4, (0.09, 0.25), 12345, 4)
    assert np.array_equal(a, b)
    assert not np.array_equal(a, c)
    e = O.sample_perturbations(100000, 1, (0.09, 0.25), 12345, 0)
    mv, mw = e[:, 0, 0].mean(), e[:, 0, 1].mean()
    assert abs(mv) <= 4 * math.sqrt(0.09 / 100000)
    assert abs(mw) <= 4 * math.sqrt(0.25 / 100000)


# ---------------------------------------------------------------- core / dynamics
def test_wrap_angle():  # test_core.cpp:12-19, test_smoke.py:12-15
    L = O.lib()
    assert L.orc_wrap_angle(0.0) == 0.0
    assert L.orc_wrap_angle(-math.pi) == pytest.approx(math.pi)
    assert L.orc_wrap_angle(3 * math.pi) == pytest.approx(math.pi)
    assert L.orc_wrap_angle(math.pi) == pytest.approx(math.pi)


def step(s, u):
    out = np.empty(5)
    O.lib().orc_step_nominal(P(f(s)), P(f(u)), NOM, P(out))
    return out


def jac(s, u):
    J = np.empty(25)
    O.lib().orc_jacobian_nominal(P(f(s)), P(f(u)), NOM, P(J))
    return J.reshape(5, 5)


def test_step_nominal_worked_examples():  # test_dynamics.cpp:39-60
    n = step([0, 0, 0, 0, 0], [0, 0])
    assert n[0] == 0 and n[1] == 0 and n[3] == 0 and n[4] == 0
    n = step([0, 0, 0, 1, 0], [1, 0])
    assert n[3] == pytest.approx(1.0) and n[0] == pytest.approx(0.05) and n[1] == pytest.approx(0)
    n = step([0, 0, 0, 0, 0], [2, 0])
    assert n[3] == pytest.approx(0.2) and n[0] == pytest.approx(0.0)


def test_lag_contraction_and_chord():  # test_dynamics.cpp:62-89
    rng = np.random.default_rng(3)
    for _ in range(100):
        s = [rng.uniform(-5, 5), rng.uniform(-5, 5), rng.uniform(-3, 3), rng.uniform(-0.5, 2),
             rng.uniform(-2, 2)]
        u = [rng.uniform(-0.5, 2), rng.uniform(-2, 2)]
        n = step(s, u)
        assert abs(n[3] - u[0]) == pytest.approx((1 - 0.1) * abs(s[3] - u[0]), rel=1e-12)
        n0 = step(s, [0, 0])
        assert math.hypot(n0[0] - s[0], n0[1] - s[1]) <= abs(s[3]) * 0.05 + 1e-12


def test_jacobian_closed_forms_and_fd():  # test_dynamics.cpp:91-117
    J = jac([1, 2, 0.3, 1.0, 0.2], [1, 0])
    assert J[3, 3] == pytest.approx(0.9) and J[4, 4] == pytest.approx(1 - 0.05 / 0.35)
    J = jac([0, 0, 0.7, 1.0, 0.0], [1, 0])
    assert J[0, 3] == pytest.approx(0.05 * math.cos(0.7), rel=1e-9)
    assert J[1, 3] == pytest.approx(0.05 * math.sin(0.7), rel=1e-9)
    rng = np.random.default_rng(17)
    for _ in range(100):
        s = np.array([rng.uniform(-5, 5), rng.uniform(-5, 5), rng.uniform(-3, 3),
                      rng.uniform(-0.5, 2), rng.uniform(-2, 2)])
        u = [rng.uniform(-0.5, 2), rng.uniform(-2, 2)]
        J = jac(s, u)
        Jfd = np.empty((5, 5))
        h = 1e-6
        for c in range(5):
            hi, lo = s.copy(), s.copy()
            hi[c] += h
            lo[c] -= h
            d = step(hi, u) - step(lo, u)
            d[2] = math.remainder(d[2], 2 * math.pi)
            Jfd[:, c] = d / (2 * h)
        scale = max(1.0, np.abs(Jfd).max())
        assert np.abs(J - Jfd).max() / scale <= 1e-6


def test_kinematic_and_edd5():  # test_dynamics.cpp:119-160
    L = O.lib()
    out = np.empty(5)
    L.orc_step_kinematic(P(f([1, 1, 0.5, 0.7, 0.1])), P(f([0, 0])), 1.0, P(out))
    assert out[0] == 1 and out[1] == 1 and out[3] == 0 and out[4] == 0
    L.orc_step_kinematic(P(f([0, 0, 0, 0, 0])), P(f([math.pi, math.pi])), 1.0, P(out))
    assert out[0] == pytest.approx(0, abs=1e-12) and out[1] == pytest.approx(2.0)
    assert out[2] == pytest.approx(math.pi)
    width = 0.37
    ideal = O.Edd5(1.0, 1.0, 0.0, -0.5 * width, 0.5 * width)
    rng = np.random.default_rng(23)
    for _ in range(200):
        s = f([rng.uniform(-5, 5), rng.uniform(-5, 5), rng.uniform(-3, 3), rng.uniform(-0.5, 2),
               rng.uniform(-2, 2)])
        u = f([rng.uniform(-0.5, 2), rng.uniform(-2, 2)])
        a, b = np.empty(5), np.empty(5)
        L.orc_step_edd5(P(s), P(u), ideal, width, 0.05, P(a))
        L.orc_step_kinematic(P(s), P(u), 0.05, P(b))
        assert np.abs(a - b).max() <= 1e-12
    slip = O.Edd5(0.9, 0.9, 0.0, -0.5 * width, 0.5 * width)
    L.orc_step_edd5(P(f([0, 0, 0, 0, 0])), P(f([1.5, 0])), slip, width, 0.05, P(a))
    assert a[3] == pytest.approx(0.9 * 1.5) and a[4] == pytest.approx(0.0)


# ---------------------------------------------------------------- gp.cpp
def kp(sv=1.0, ls=(1, 1, 1, 1), nv=1e-4):
    return [sv, *ls, nv]


def random_inputs(rng, n):
    return np.column_stack([rng.uniform(-0.5, 2, n), rng.uniform(-2, 2, n),
                            rng.uniform(-0.5, 2, n), rng.uniform(-2, 2, n)])


def test_kernel_closed_forms():  # test_gp.cpp:48-63
    L = O.lib()
    a = f([0.3, -0.2, 1.0, 0.5])
    assert L.orc_kernel_eval(P(a), P(a), P(f(kp(1.0)))) == pytest.approx(1.0)
    b = a.copy()
    b[0] += 0.7
    k = f(kp(2.0, (0.7, 1, 1, 1)))
    assert L.orc_kernel_eval(P(a), P(b), P(k)) == pytest.approx(2 * math.exp(-0.5), rel=1e-12)


def test_single_point_closed_form():  # test_gp.cpp:65-78, test_smoke.py:37-48
    g = O.GP(np.zeros((1, 4)), np.array([[2.0]]), [kp(1.0, nv=1.0)])
    m, v = g.predict_batch(np.zeros((3, 4)))
    np.testing.assert_allclose(m[:, 0], 1.0, rtol=1e-12)
    np.testing.assert_allclose(v[:, 0], 0.5, rtol=1e-12)


def test_prior_recovery():  # test_gp.cpp:80-92
    rng = np.random.default_rng(2)
    x = random_inputs(rng, 32)
    y = rng.standard_normal((32, 1))
    g = O.GP(x, y, [kp(1.7, nv=1e-2)])
    m, v = g.predict_batch(np.full((1, 4), 500.0))
    assert abs(m[0, 0]) <= 1e-10 and v[0, 0] == pytest.approx(1.7, rel=1e-10)


def test_predict_matches_dense_inverse():  # test_gp.cpp:94-122
    rng = np.random.default_rng(5)
    for _ in range(20):
        n = 8 + int(rng.uniform(0, 56))
        x = random_inputs(rng, n)
        y = np.column_stack([np.sin(x[:, 0]) + 0.1 * rng.standard_normal(n),
                             0.3 * x[:, 1] + 0.1 * rng.standard_normal(n)])
        k = kp(rng.uniform(0.2, 2), tuple(rng.uniform(0.3, 2, 4)), rng.uniform(1e-4, 1e-2))
        g = O.GP(x, y, [k, k])
        ls = np.array(k[1:5])
        Kxx = k[0] * np.exp(-0.5 * (((x[:, None, :] - x[None, :, :]) / ls) ** 2).sum(-1))
        Kinv = np.linalg.inv(Kxx + k[5] * np.eye(n))
        q = random_inputs(rng, 3)
        m, v = g.predict_batch(q)
        for i in range(3):
            ks = k[0] * np.exp(-0.5 * (((x - q[i]) / ls) ** 2).sum(-1))
            for j in range(2):
                assert abs(m[i, j] - ks @ Kinv @ y[:, j]) <= 1e-8
                assert abs(v[i, j] - max(k[0] - ks @ Kinv @ ks, 0)) <= 1e-8


def test_batch_equals_single_and_groups():  # test_gp.cpp:157-183
    rng = np.random.default_rng(13)
    x = random_inputs(rng, 100)
    y = np.column_stack([np.sin(x[:, 0]), np.cos(x[:, 1]), 0.2 * x[:, 2]])
    shared = kp(0.5, nv=1e-4)
    other = kp(0.5, (2, 2, 2, 2), 1e-4)
    g = O.GP(x, y, [shared, shared, other])
    assert g.n_groups() == 2
    q = random_inputs(rng, 256)
    mb, vb = g.predict_batch(q)
    for i in (0, 1, 17, 100, 255):
        ms, vs = g.predict_batch(q[i:i + 1])
        assert np.abs(mb[i] - ms[0]).max() <= 1e-12 and np.abs(vb[i] - vs[0]).max() <= 1e-12


def test_factor_and_jitter():  # test_gp.cpp:185-220
    rng = np.random.default_rng(15)
    x = random_inputs(rng, 40)
    g = O.GP(x, rng.standard_normal((40, 1)), [kp(1.3, nv=1e-3)])
    gr = g.group(0)
    ls = np.ones(4)
    Kxx = 1.3 * np.exp(-0.5 * (((x[:, None, :] - x[None, :, :]) / ls) ** 2).sum(-1))
    Kxx += (1e-3 + g.jitter(0)) * np.eye(40)
    Lc = gr["chol"]
    assert np.linalg.norm(Lc @ Lc.T - Kxx) / np.linalg.norm(Kxx) <= 1e-8
    np.testing.assert_allclose(gr["inv_lower_t"].T @ Lc, np.eye(40), atol=1e-8)
    dup = np.ones((2, 4))
    try:
        gd = O.GP(dup, np.ones((2, 1)), [kp(1.0, nv=1e-300)])
        assert 0 < gd.jitter(0) <= 1e-6
    except RuntimeError as e:
        assert "jitter" in str(e)


def test_fit_validation():  # test_gp.cpp:222-231
    with pytest.raises(ValueError):
        O.GP(np.random.rand(3, 4), np.random.rand(3, 1), [kp(-1.0)])


def test_ensemble_combine():  # test_gp.cpp:283-321
    L = O.lib()
    means = f([[1, 0], [-1, 0], [0, 0]])
    vars_ = f([[0.3, 0.2]] * 3)
    out_m, out_c = np.empty(2), np.empty(2)
    assert L.orc_ensemble_combine(P(means), P(vars_), P(f([1, 0, 0])), 3, P(out_m), P(out_c)) == 0
    assert out_m[0] == 1.0 and out_c[0] == 0.3 and out_c[1] == 0.2
    L.orc_ensemble_combine(P(means), P(vars_), P(f([1 / 3] * 3)), 3, P(out_m), P(out_c))
    assert out_c[0] == pytest.approx(0.1, rel=1e-12) and out_c[1] == pytest.approx(0.2 / 3, rel=1e-12)
    L.orc_ensemble_combine(P(means), P(vars_), P(f([0.5, 0.5, 0])), 3, P(out_m), P(out_c))
    assert out_m[0] == 0.0 and out_m[1] == 0.0
    assert L.orc_ensemble_combine(P(means), P(vars_), P(f([0.6, 0.6, 0])), 3, P(out_m), P(out_c)) == 1


# ---------------------------------------------------------------- uncertainty.cpp
def test_quantiles():  # test_uncertainty.cpp:45-74, test_smoke.py:18-21
    L = O.lib()
    assert L.orc_chi2_quantile_2dof(0.0) == 0.0
    assert L.orc_chi2_quantile_2dof(0.5) == pytest.approx(1.3862943611198906, rel=1e-12)
    assert L.orc_chi2_quantile_2dof(0.95) == pytest.approx(5.991464547107979, rel=1e-12)
    assert L.orc_normal_quantile(0.5) == pytest.approx(0.0, abs=1e-12)
    assert L.orc_normal_quantile(0.975) == pytest.approx(1.959963984540054, rel=1e-9)
    assert L.orc_normal_quantile(0.95) == pytest.approx(1.6448536269514722, rel=1e-9)
    for p in (0.6, 0.8, 0.95, 0.99):
        assert abs(L.orc_normal_cdf(L.orc_normal_quantile(p)) - p) <= 1e-9


def test_lambda_max():  # test_uncertainty.cpp:76-86
    L = O.lib()
    assert L.orc_lambda_max_2x2(P(f([0.02, 0, 0, 0.01]))) == pytest.approx(0.02, rel=1e-15)
    rng = np.random.default_rng(3)
    for _ in range(200):
        a = rng.uniform(-1, 1, (2, 2))
        s = a @ a.T
        assert L.orc_lambda_max_2x2(P(f(s.ravel()))) == pytest.approx(np.linalg.eigvalsh(s).max(),
                                                                       rel=1e-10, abs=1e-14)


def test_belief_propagation_basics():  # test_uncertainty.cpp:88-113
    L = O.lib()
    mu = f([0, 0, 0, 1.0, 0.2])
    om, oc = np.empty(5), np.empty(25)
    L.orc_propagate_belief(P(mu), P(np.zeros(25)), P(f([1, 0])), P(f([0, 0])), P(f([0, 0])), NOM,
                           P(om), P(oc))
    assert np.linalg.norm(oc) == 0.0
    L.orc_propagate_belief(P(mu), P(np.zeros(25)), P(f([1, 0])), P(f([0, 0])),
                           P(f([0.04, 0.09])), NOM, P(om), P(oc))
    C = oc.reshape(5, 5)
    assert C[3, 3] == pytest.approx(0.04) and C[4, 4] == pytest.approx(0.09)
    assert np.linalg.norm(C[:3, :3]) == 0.0
    L.orc_propagate_belief(P(mu), P(np.zeros(25)), P(f([1, 0])), P(f([0.1, -0.05])),
                           P(f([0, 0])), NOM, P(om), P(oc))
    nn = step(mu, [1, 0])
    assert om[3] == pytest.approx(nn[3] + 0.1) and om[4] == pytest.approx(nn[4] - 0.05)


def test_tightening_closed_forms():  # test_uncertainty.cpp:171-213, test_smoke.py:71-80
    L = O.lib()
    chi2 = L.orc_chi2_quantile_2dof(0.95)
    assert L.orc_tighten_lane_radius(1.0, P(np.zeros(4)), chi2) == pytest.approx(1.0)
    r = L.orc_tighten_lane_radius(1.0, P(f([0.01, 0, 0, 0.01])), chi2)
    assert r == pytest.approx(1 - math.sqrt(5.991464547107979 * 0.01), rel=1e-9)
    assert 1 - r == pytest.approx(0.24478, rel=1e-4)
    r = L.orc_tighten_lane_radius(1.0, P(f([0.02, 0, 0, 0.01])), chi2)
    assert r == pytest.approx(1 - math.sqrt(5.991464547107979 * 0.02), rel=1e-9)
    assert L.orc_tighten_lane_radius(0.1, P(f([1, 0, 0, 1])), chi2) < 0
    z = L.orc_normal_quantile(0.975)
    import ctypes as C
    d = C.c_double()
    deg = C.c_int()
    nrm = np.empty(2)
    dbar = L.orc_tighten_obstacle_distance(P(f([2, 0])), P(f([0, 0])), 1.0, P(np.zeros(4)), z,
                                           C.byref(d), P(nrm), C.byref(deg))
    assert d.value == pytest.approx(1.0) and dbar == pytest.approx(1.0)
    dbar = L.orc_tighten_obstacle_distance(P(f([2, 0])), P(f([0, 0])), 1.0,
                                           P(f([0.01, 0, 0, 0.01])), z, C.byref(d), P(nrm),
                                           C.byref(deg))
    assert dbar == pytest.approx(1 - 1.959963984540054 * 0.1, rel=1e-9)
    assert dbar == pytest.approx(0.80400, rel=1e-4)
    dbar = L.orc_tighten_obstacle_distance(P(f([0, 0])), P(f([0, 0])), 0.5,
                                           P(f([0.01, 0, 0, 0.01])), z, C.byref(d), P(nrm),
                                           C.byref(deg))
    assert deg.value == 1 and tuple(nrm) == (1.0, 0.0) and d.value == pytest.approx(-0.5)


# ---------------------------------------------------------------- costs.cpp
def cdist(t, x, y):
    return O.lib().orc_centerline_distance(t, x, y)


def test_lane_geometry():  # test_costs.cpp:27-58
    c = O.make_track("circle", (0, 0), 10.0, 1.0)
    assert cdist(c, 10, 0) == pytest.approx(0.0) and cdist(c, 11, 0) == pytest.approx(1.0)
    assert cdist(c, 12, 0) / 1.0 == pytest.approx(2.0)
    p = O.make_track("poly", half_width=0.5, waypoints=[[0, 0], [10, 0], [10, 10]], closed=False)
    assert cdist(p, 5, 0) == pytest.approx(0.0) and cdist(p, 5, 0.5) / 0.5 == pytest.approx(1.0)
    assert cdist(p, 10.25, 5.0) / 0.5 == pytest.approx(0.5)
    assert abs(cdist(p, 9.99, 0.3) - cdist(p, 10.01, 0.3)) <= 0.05
    sq = O.make_track("poly", half_width=0.5, waypoints=[[0, 0], [4, 0], [4, 4], [0, 4]], closed=True)
    assert cdist(sq, 0, 2) == pytest.approx(0.0)
    # inclusive violation boundary: 11.0 → not violated at r_bar = 1
    assert not (cdist(c, 11.0, 0) > 1.0)
    assert cdist(c, 11.0001, 0) > 1.0
    assert cdist(c, 10.8, 0) > 0.5


def test_slip_ratio():  # test_costs.cpp:60-76
    L = O.lib()
    assert L.orc_slip_ratio(P(f([0, 0, 0, 1, 0])), P(f([0.05, 0, 0, 1, 0]))) == 0.0
    a = f([0, 0, 0, 2.0, 1.0])
    b = step(a, [2, 1])
    assert L.orc_slip_ratio(P(a), P(b)) == pytest.approx(math.tan(0.025), rel=1e-9)
    a = f([1, 1, 0.5, 0, 0])
    assert L.orc_slip_ratio(P(a), P(a)) == 0.0


def test_collision_and_goal():  # test_costs.cpp:78-99
    L = O.lib()
    obs = f([[0, 0, 1.0], [5, 0, 0.5]])
    assert L.orc_collision_indicator(3, 3, None, 0, None) == 0.0
    assert L.orc_collision_indicator(0.5, 0, P(obs), 2, P(np.zeros(2))) == 1.0
    assert L.orc_collision_indicator(1.5, 0, P(obs), 2, P(np.zeros(2))) == 0.0
    assert L.orc_collision_indicator(1.5, 0, P(obs), 2, P(f([0.6, 0]))) == 1.0


def straight(n, v=2.0, dt=0.05):
    return f([[v * dt * k, 0, 0, v, 0] for k in range(n + 1)])


def test_tracking_cost_structure():  # test_costs.cpp:101-154
    L = O.lib()
    track = O.make_track("poly", half_width=0.5, waypoints=[[-100, 0], [100, 0]], closed=False)
    n = 10
    st = straight(n)
    tr = np.zeros(n)
    rb = np.full(n, 0.5)
    vs = np.full(n, 2.0)

    def cost(w, states=st, trace=tr, rbar=rb, vsam=vs, nn=n):
        return L.orc_tracking_cost(P(states), P(trace), nn, track, P(rbar), 2.0, P(vsam),
                                   O.TrackingWeights(*w))
    assert cost((0, 0, 0, 0, 0)) == 0.0
    assert cost((0.5, 1, 0, 1, 0.5)) <= 1e-12
    assert cost((0, 0, 0, 0, 1), vsam=np.full(n, 1.5)) == pytest.approx(n * 0.5, rel=1e-12)
    assert cost((0, 0, 0, 0, 1), vsam=np.full(n, 2.5)) == 0.0
    assert cost((1, 0, 0, 0, 0), trace=np.full(n, 0.03)) == pytest.approx(n * 0.03, rel=1e-12)
    nn = 12
    s12 = straight(nn)

    def viol(k):
        s2 = s12.copy()
        s2[k + 1, 1] = 2.0
        return cost((0, 0, 0, 1, 0), states=s2, trace=np.zeros(nn), rbar=np.full(nn, 0.5),
                    vsam=np.full(nn, 2.0), nn=nn)
    assert viol(10) / viol(0) == pytest.approx(0.9 ** 10, rel=1e-12)


def test_avoidance_cost_structure():  # test_costs.cpp:156-189
    L = O.lib()
    goal = f([2.0, 0.0, 0.3])
    n = 8
    st = straight(n)
    obs = f([[0.2, 0.0, 0.05]])
    m = np.zeros((n, 1))
    aw = lambda *w: O.AvoidanceWeights(*w)  # noqa: E731
    assert L.orc_avoidance_cost(P(st), P(np.zeros(n)), n, P(obs), 1, P(m), P(goal),
                                aw(0, 0, 0, 0), 1e4) == 0.0
    c = L.orc_avoidance_cost(P(st), P(np.zeros(n)), n, None, 0, None, P(goal), aw(0, 1, 1, 1), 1e4)
    assert c == pytest.approx(1e4 + sum(abs(2 - 0.1 * k) for k in range(1, n + 1)), rel=1e-12)
    assert L.orc_avoidance_cost(P(st), P(np.zeros(n)), n, P(obs), 1, P(m), P(goal),
                                aw(0, 1, 0, 0), 1e4) == pytest.approx(1.0)


# ---------------------------------------------------------------- mppi.cpp
def tw(costs, lam):
    c = f(costs)
    w = np.empty(len(c))
    O.lib().orc_trajectory_weights(P(c), len(c), lam, P(w))
    return w


def test_trajectory_weights():  # test_mppi.cpp:70-117
    w = tw(np.full(8, 3.0), 0.5)
    assert w.sum() == pytest.approx(1.0, rel=1e-12) and np.allclose(w, 0.125, rtol=1e-12)
    w = tw([0.0, 0.1], 0.1)
    z = 1 + math.exp(-1)
    assert w[0] == pytest.approx(1 / z, rel=1e-12) and w[1] == pytest.approx(math.exp(-1) / z, rel=1e-12)
    assert tw([5.0, 1.0, 9.0], 1e-6)[1] == pytest.approx(1.0, rel=1e-9)
    a = tw([1, 2, 3, 4], 0.7)
    b = tw(np.array([1, 2, 3, 4]) + 1e6, 0.7)
    assert np.abs(a - b).max() <= 1e-12
    w = tw([1.0, np.inf, np.nan], 0.5)
    assert w[0] == pytest.approx(1.0) and w[1] == 0 and w[2] == 0
    assert np.abs(tw([np.nan] * 3, 0.5)).max() == 0.0
    rng = np.random.default_rng(5)
    for _ in range(50):
        c = rng.uniform(0, 10, 32)
        assert tw(c, 0.3) @ c <= c.mean() + 1e-12


def test_update_and_shift():  # test_mppi.cpp:119-160
    L = O.lib()
    lo, hi = f([-0.5, -2]), f([2, 2])
    nom = f([[1.0, 0.0]] * 3)
    out = np.empty((3, 2))
    e1 = np.zeros((1, 3, 2))
    e1[0, 1, 0] = 0.3
    L.orc_update_controls(P(nom), P(e1), P(f([1.0])), 1, 3, P(lo), P(hi), P(out))
    assert out[1, 0] == pytest.approx(1.3)
    e1 = np.full((1, 3, 2), 100.0)
    L.orc_update_controls(P(nom), P(e1), P(f([1.0])), 1, 3, P(lo), P(hi), P(out))
    assert out[0, 0] == 2.0 and out[0, 1] == 2.0
    seq = f([[1, 0], [2, 0], [3, 0]])
    s1 = np.empty((3, 2))
    L.orc_shift_horizon(P(seq), 3, P(s1))
    assert s1[0, 0] == 2 and s1[2, 0] == 3
    s2 = np.empty((3, 2))
    L.orc_shift_horizon(P(s1), 3, P(s2))
    assert (s2[:, 0] == 3).all()


def zero_residual_gp(R, noise=1e-6):  # test_mppi.cpp:13-24 (restated sampling of inputs)
    rng = O.lib()
    r = np.random.default_rng(77)
    x = random_inputs(r, 24)
    return O.GP(x, np.zeros((24, 2 * R)), [kp(1.0, nv=noise)] * (2 * R))


def test_planner_thread_count_bit_identity():  # test_mppi.cpp:231-258
    gp = zero_residual_gp(2, 1e-4)
    track = O.make_track("circle", (0, 0), 2.0, 0.4)
    task = O.make_task(O.ORC_TASK_TRACKING, track, 1.5)

    def run(threads):
        p = O.Planner(300, 10, gp=gp, n_terrains=2, seed=12345, threads=threads, p_x=0.9)
        s = np.array([2.0, 0.0, 1.57, 0.5, 0.0])
        cmds = []
        for _ in range(5):
            c, _ = p.plan_step(s, task)
            cmds.append(c)
            s = step(s, c)
        return np.array(cmds)
    a, b, c = run(1), run(8), run(1)
    assert np.array_equal(a, b) and np.array_equal(a, c)


def test_degenerate_planner_identity():  # test_mppi.cpp:260-276
    gp = zero_residual_gp(1, 1e-4)
    p = O.Planner(1, 5, gp=gp, n_terrains=1, sigma_sim=(1e-18, 1e-18), threads=1, p_x=0.9)
    lane = O.make_track("poly", half_width=0.5, waypoints=[[-10, 0], [10, 0]], closed=False)
    task = O.make_task(O.ORC_TASK_TRACKING, lane, 0.0)
    c, _ = p.plan_step(np.zeros(5), task)
    assert abs(c[0]) <= 1e-8 and abs(c[1]) <= 1e-8


def test_tightening_monotone_radii():  # test_mppi.cpp:278-311
    r = np.random.default_rng(23)
    x = random_inputs(r, 40)
    y = 0.02 * r.standard_normal((40, 2))
    gp = O.GP(x, y, [kp(4e-4, nv=1e-5)] * 2)
    p = O.Planner(32, 12, gp=gp, n_terrains=1, seed=12345, threads=1, p_x=0.95)
    lane = O.make_track("poly", half_width=0.5, waypoints=[[-100, 0], [100, 0]], closed=False)
    task = O.make_task(O.ORC_TASK_TRACKING, lane, 1.0)
    p.plan_step(np.array([0, 0, 0, 1.0, 0]), task)
    rb = p.lane_radii()
    assert rb[0] == 0.5 and rb[11] < 0.5
    assert all(rb[k] <= rb[k - 1] + 1e-12 for k in range(1, 12))
    cov = p.horizon_covariances()
    assert cov[-1, 0, 0] >= cov[0, 0, 0]


def test_first_tick_margins_nonnegative():  # test_mppi.cpp:313-325
    gp = zero_residual_gp(1, 1e-4)
    p = O.Planner(4, 6, gp=gp, n_terrains=1, seed=12345, threads=1, p_x=0.95)
    task = O.make_task(O.ORC_TASK_AVOIDANCE, obstacles=[[3, 0, 0.5]], goal=(6, 0, 0.5))
    p.plan_step(np.zeros(5), task)
    m = p.obstacle_margins()
    assert m.shape == (6, 1) and m.min() >= 0.0


def test_config_validation():  # test_mppi.cpp:327-337
    with pytest.raises(ValueError):
        O.Planner(0, 5, model_kind=O.ORC_MODEL_UNICYCLE)
    with pytest.raises(ValueError):
        O.Planner(4, 5, model_kind=O.ORC_MODEL_UNICYCLE, lam=0.0)
    with pytest.raises(ValueError):
        O.Planner(4, 5, model_kind=O.ORC_MODEL_UNICYCLE, lo=(3.0, -2.0))


def test_zero_residual_planner_first_step_matches_scalar_path():  # test_mppi.cpp:181-229
    r = np.random.default_rng(17)
    n, m = 60, 2
    x = random_inputs(r, n)
    y = np.empty((n, 2 * m))
    for t in range(m):
        y[:, 2 * t] = 0.02 * np.sin(x[:, 0] + t) + 0.01 * x[:, 2]
        y[:, 2 * t + 1] = -0.015 * x[:, 3] + 0.005 * t
    gp = O.GP(x, y, [kp(0.01, nv=1e-5)] * (2 * m))
    p = O.Planner(257, 6, gp=gp, n_terrains=m, seed=12345, threads=1, p_x=0.95)
    p.set_terrain_weights([0.3, 0.7])
    track = O.make_track("circle", (0, 0), 2.0, 0.4)
    task = O.make_task(O.ORC_TASK_TRACKING, track, 1.5)
    x0 = np.array([2.0, 0.0, 1.5707963267948966, 1.0, 0.5])
    p.plan_step(x0, task)
    assert np.isfinite(p.costs()).all()
    assert p.weights().sum() == pytest.approx(1.0, rel=1e-12)


def test_zero_residual_rollout_equals_nominal():  # test_mppi.cpp:162-179
    gp = zero_residual_gp(3)
    r = np.random.default_rng(9)
    seq = np.column_stack([r.uniform(0, 2, 10), r.uniform(-1, 1, 10)])
    x0 = np.array([0.0, 0.0, 0.3, 1.0, 0.2])
    states, corr = O.rollout(x0, seq, O.ORC_MODEL_GP, gp, 3, [1 / 3] * 3)
    s = x0.copy()
    for k in range(10):
        nxt = np.empty(5)
        O.lib().orc_step_nominal(P(s), P(f(seq[k])), O.Nominal(0.5, 0.35, 0.05), P(nxt))
        s = nxt
        assert abs(states[k + 1, 0] - s[0]) <= 1e-9 and abs(states[k + 1, 3] - s[3]) <= 1e-9
        assert np.abs(corr[k, :2]).max() <= 1e-9
    with pytest.raises(ValueError):
        O.rollout(x0, seq, O.ORC_MODEL_GP, gp, 3, [0.5, 0.5, 0.5])
    st_k, _ = O.rollout(x0, seq, O.ORC_MODEL_UNICYCLE)
    assert st_k.shape == (11, 5) and np.isfinite(st_k).all()
