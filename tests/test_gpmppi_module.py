"""The reference's Python module surface (`import gpmppi`, bindings/module.cpp:40-219).

The ten cases restate /root/reference/proj/tests/python/test_smoke.py:12-122 against the
repository's `gpmppi` package; the host-only ones run on CPU, the GP and closed-loop ones
on the GPU. When the reference tree is present (this container) its own test file is also
run in place for the CPU-only cases (it needs a GPU for the rest; see profiles/r02).
"""
import json
import math
import os
import subprocess
import sys
import tempfile

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SMOKE = "/root/reference/proj/tests/python/test_smoke.py"

gpmppi = pytest.importorskip("gpmppi")


def test_wrap_angle():  # test_smoke.py:12-15
    assert gpmppi.wrap_angle(0.0) == 0.0
    assert gpmppi.wrap_angle(3 * math.pi) == pytest.approx(math.pi)
    assert gpmppi.wrap_angle(-math.pi) == pytest.approx(math.pi)


def test_quantiles():  # test_smoke.py:18-21
    assert gpmppi.chi2_quantile_2dof(0.95) == pytest.approx(-2 * math.log(0.05))
    assert gpmppi.normal_quantile(0.975) == pytest.approx(1.959964, abs=1e-5)
    assert gpmppi.normal_cdf(gpmppi.normal_quantile(0.8)) == pytest.approx(0.8, abs=1e-9)
    with pytest.raises(ValueError):
        gpmppi.normal_quantile(1.0)
    with pytest.raises(ValueError):
        gpmppi.chi2_quantile_2dof(1.0)


def test_dynamics_step():  # test_smoke.py:24-35
    p = gpmppi.NominalParams(tau_v=0.5, tau_omega=0.35, dt=0.05)
    nxt = gpmppi.step_nominal(np.zeros(5), np.array([2.0, 0.0]), p)
    assert nxt[3] == pytest.approx(0.2)
    uni = gpmppi.step_kinematic_unicycle(np.zeros(5), np.array([1.0, 0.0]), 1.0)
    assert uni[0] == pytest.approx(1.0)
    jac = gpmppi.jacobian_nominal(np.array([0.0, 0.0, 0.0, 1.0, 0.1]), np.array([1.0, 0.0]), p)
    assert jac.shape == (5, 5)
    assert jac[3, 3] == pytest.approx(0.9)
    with pytest.raises(ValueError):
        gpmppi.NominalParams(tau_v=0.5, tau_omega=0.35, dt=0.5)
    with pytest.raises(ValueError):
        gpmppi.step_nominal(np.array([np.nan, 0, 0, 0, 0]), np.zeros(2), p)


def test_jacobian_matches_finite_differences():  # test_dynamics.cpp FD check, host C++ path
    p = gpmppi.NominalParams()
    s, u = np.array([0.3, -0.2, 0.7, 1.1, 0.4]), np.array([1.2, -0.3])
    J = gpmppi.jacobian_nominal(s, u, p)
    h = 1e-6
    for j in range(5):
        e = np.zeros(5)
        e[j] = h
        fd = (gpmppi.step_nominal(s + e, u, p) - gpmppi.step_nominal(s - e, u, p)) / (2 * h)
        np.testing.assert_allclose(J[:, j], fd, atol=1e-6)


def test_simplex_projection():  # test_smoke.py:78-82
    np.testing.assert_allclose(gpmppi.project_simplex(np.array([2.0, 0.0, 0.0])), [1.0, 0.0, 0.0])
    np.testing.assert_allclose(gpmppi.project_simplex(np.array([0.5, 0.5, 0.5])), [1 / 3] * 3, atol=1e-12)


def test_tightening():  # test_smoke.py:85-94
    r = gpmppi.tighten_lane_radius(1.0, 0.01 * np.eye(2), p_x=0.95)
    assert r == pytest.approx(1.0 - math.sqrt(-2 * math.log(0.05) * 0.01), abs=1e-9)
    d_bar, normal, degenerate = gpmppi.tighten_obstacle_distance(
        np.array([2.0, 0.0]), np.array([0.0, 0.0]), 1.0, 0.01 * np.eye(2), p_x=0.975)
    assert d_bar == pytest.approx(0.80400, abs=1e-4)
    assert not degenerate
    np.testing.assert_allclose(np.linalg.norm(normal), 1.0)
    _, n2, deg2 = gpmppi.tighten_obstacle_distance(np.zeros(2), np.zeros(2), 1.0, np.eye(2))
    assert deg2 and list(n2) == [1.0, 0.0]  # uncertainty.cpp:105-108


def test_default_config_is_json():  # test_smoke.py:97-100
    cfg = json.loads(gpmppi.default_config_json())
    assert cfg["mppi"]["samples"] == 1024
    assert cfg["scenario"]["kind"] == "tracking"


def test_config_loader_rejects_unknown_keys(tmp_path):  # config.cpp:40-46
    from paper_2411_03289_b200 import config as CF
    cfg = json.loads(gpmppi.default_config_json())
    cfg["mppi"]["sample"] = 3
    p = tmp_path / "c.json"
    p.write_text(json.dumps(cfg))
    with pytest.raises(ValueError, match=r"unknown key '\$\.mppi\.sample'"):
        CF.load_config(str(p))
    cfg = json.loads(gpmppi.default_config_json())
    cfg["gp"] = {"hyperparams": "grid", "signal_var": 1.0}
    p.write_text(json.dumps(cfg))
    with pytest.raises(ValueError, match="only allowed with hyperparams=fixed"):
        CF.load_config(str(p))
    ok = json.loads(gpmppi.default_config_json())
    ok["scenario"]["obstacles"] = [[1.0, 2.0, 0.3]]
    del ok["scenario"]["random_obstacles"]
    p.write_text(json.dumps(ok))
    back = CF.load_config(str(p))
    assert back["scenario"]["obstacles"] == [[1.0, 2.0, 0.3]] and "random_obstacles" not in back["scenario"]
    assert CF.load_config(str(p)) == back and len(CF.config_hash_hex(back)) == 16


def test_kernel_and_combine():
    k = gpmppi.KernelParams(2.0, np.ones(4), 1.0)
    assert gpmppi.kernel_eval(np.zeros(4), np.zeros(4), k) == pytest.approx(2.0)  # test_gp.cpp:48-63
    assert gpmppi.kernel_eval(np.zeros(4), np.array([1.0, 0, 0, 0]), k) == pytest.approx(2 * math.exp(-0.5))
    mean, cov = gpmppi.ensemble_combine(np.array([[1.0, 2.0], [3.0, 4.0]]), np.ones((2, 2)), np.array([0.25, 0.75]))
    np.testing.assert_allclose(mean, [2.5, 3.5])
    np.testing.assert_allclose(cov, np.diag([0.625, 0.625]))
    with pytest.raises(ValueError):
        gpmppi.ensemble_combine(np.ones((2, 2)), np.ones((2, 2)), np.array([0.5, 0.6]))
    with pytest.raises(ValueError):
        gpmppi.KernelParams(0.0, np.ones(4), 1.0)


@pytest.mark.skipif(not os.path.exists(REF_SMOKE), reason="reference tree not present (GPU box)")
def test_reference_smoke_file_in_place_host_cases():
    """The reference's own test file, run in place against this package (host-only cases)."""
    env = {**os.environ, "PYTHONPATH": ROOT}
    r = subprocess.run([sys.executable, "-m", "pytest", REF_SMOKE, "-q", "-p", "no:cacheprovider",
                        "--rootdir", tempfile.gettempdir(), "-k", "not gp_ and not tracking and not unicycle"],
                       capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "6 passed" in r.stdout


@pytest.mark.gpu
def test_gp_single_point_closed_form():  # test_smoke.py:38-50
    model = gpmppi.GpModel.fit(np.zeros((1, 4)), np.array([[2.0]]), [gpmppi.KernelParams(1.0, np.ones(4), 1.0)])
    mean, var = model.predict(np.zeros(4))
    assert mean[0] == pytest.approx(1.0)
    assert var[0] == pytest.approx(0.5)
    bmean, bvar = model.predict_batch(np.zeros((3, 4)))
    assert bmean.shape == (3, 1)
    np.testing.assert_allclose(bmean[:, 0], 1.0)
    np.testing.assert_allclose(bvar[:, 0], 0.5)
    assert model.n_points == 1 and model.n_outputs == 1


@pytest.mark.gpu
def test_gp_save_load_roundtrip(tmp_path):  # test_smoke.py:53-64
    rng = np.random.default_rng(0)
    x = rng.uniform(-1, 1, size=(20, 4))
    y = np.sin(x[:, :1])
    model = gpmppi.GpModel.fit(x, y, [gpmppi.KernelParams(0.5, np.full(4, 0.8), 1e-4)])
    path = str(tmp_path / "model.bin")
    model.save(path)
    back = gpmppi.GpModel.load(path)
    q = np.array([0.1, 0.2, 0.3, 0.4])
    np.testing.assert_array_equal(model.predict(q)[0], back.predict(q)[0])


@pytest.fixture(scope="module")
def small_config_path():  # test_smoke.py:103-123
    cfg = json.loads(gpmppi.default_config_json())
    cfg["threads"] = 1
    cfg["mppi"]["samples"] = 64
    cfg["mppi"]["horizon"] = 8
    cfg["training"] = {"n_points": 50, "hold_min": 5, "hold_max": 20}
    cfg["gp"] = {"hyperparams": "fixed", "signal_var": 4e-3, "lengthscales": [0.8, 1.2, 0.8, 1.2],
                 "noise_var": 1e-4}
    cfg["scenario"]["distance_budget"] = 3.0
    cfg["scenario"]["max_duration"] = 10.0
    with tempfile.NamedTemporaryFile("w", suffix=".json", delete=False) as f:
        json.dump(cfg, f)
        path = f.name
    yield path
    os.unlink(path)


@pytest.mark.gpu
def test_tracking_run_is_deterministic(small_config_path):  # test_smoke.py:126-132
    a = gpmppi.run_tracking(small_config_path, seed=3, planner="gp")
    b = gpmppi.run_tracking(small_config_path, seed=3, planner="gp")
    assert not a["aborted"]
    assert a["rmse"] == b["rmse"]
    assert a["ticks"] == b["ticks"]
    assert a["rmse"] < 0.5


@pytest.mark.gpu
def test_unicycle_avoidance_runs(small_config_path):  # test_smoke.py:135-138
    m = gpmppi.run_avoidance(small_config_path, seed=1, planner="unicycle")
    assert m["ticks"] > 0
    assert not m["aborted"]


@pytest.mark.gpu
def test_select_kernel_grid_and_gp_interop():
    rng = np.random.default_rng(4)
    x = rng.uniform(-1, 1, size=(60, 4))
    y = np.column_stack([0.1 * np.sin(x[:, 0]), 0.05 * x[:, 1]])
    k = gpmppi.select_kernel_grid(x, y)
    assert isinstance(k, gpmppi.KernelParams) and k.signal_var > 0
    m = gpmppi.GpModel.fit(x, y, [k, k])
    assert np.isfinite(m.log_marginal_likelihood(0))
