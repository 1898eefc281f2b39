"""Device FP64 GP factorisation (fit.cu; gp.cpp:116-138) against the host factorisation.

Both paths build the same kernel matrix; only the summation order of the Cholesky and
triangular-inverse dot products differs, so predictions agree to rounding. The device path
is the default from n = 1024; GPMPPI_FIT=host|device forces either.
"""
import os
import time

import numpy as np
import pytest

from paper_2411_03289_b200 import gpmppi as G
from paper_2411_03289_b200 import workloads as W

pytestmark = pytest.mark.gpu


def _fit(mode, X, Y, K):
    old = os.environ.get("GPMPPI_FIT")
    os.environ["GPMPPI_FIT"] = mode
    try:
        t0 = time.perf_counter()
        m = G.GpModel.fit(X, Y, K)
        return m, time.perf_counter() - t0
    finally:
        if old is None:
            del os.environ["GPMPPI_FIT"]
        else:
            os.environ["GPMPPI_FIT"] = old


@pytest.mark.parametrize("n", [37, 1100])
def test_device_fit_matches_host_fit(n):
    X, Y, K = W.gp_training_set(n, 3, seed=n)
    mh, th = _fit("host", X, Y, K)
    md, td = _fit("device", X, Y, K)
    print(f"n={n}: host fit {th * 1e3:.1f} ms, device fit {td * 1e3:.1f} ms")
    assert md.group_jitter(0) == mh.group_jitter(0)
    q = np.random.default_rng(1).uniform([-0.5, -2, -0.5, -2], [2, 2, 2, 2], size=(256, 4))
    q[:8] = X[:8]  # at training inputs the variance is smallest (most cancellation)
    mean_h, var_h = mh.predict_batch(q)
    mean_d, var_d = md.predict_batch(q)
    np.testing.assert_allclose(mean_d, mean_h, rtol=1e-8, atol=1e-11)
    np.testing.assert_allclose(var_d, var_h, rtol=0, atol=1e-10)
    for o in range(Y.shape[1]):
        lh, ld = mh.log_marginal_likelihood(o), md.log_marginal_likelihood(o)
        assert abs(ld - lh) <= 1e-9 * abs(lh)


def test_device_fit_jitter_ladder_and_failure():  # test_gp.cpp:205-220 on the device path
    X = np.ones((3, 4))
    Y = np.ones((3, 1))
    try:
        m, _ = _fit("device", X, Y, [G.KernelParams(1.0, (1, 1, 1, 1), 1e-300)])
        assert 0.0 < m.group_jitter(0) <= 1e-6
    except RuntimeError as e:
        assert "jitter" in str(e)
    with pytest.raises(RuntimeError, match="jitter"):
        _fit("device", X, Y, [G.KernelParams(1e300, (1, 1, 1, 1), 1e-300)])  # exactly singular


def test_default_fit_at_config3_size_is_device_and_fast():
    X, Y, K = W.gp_training_set(2048, 3, seed=0)
    t0 = time.perf_counter()
    m = G.GpModel.fit(X, Y, K)
    dt = time.perf_counter() - t0
    print(f"n=2048 default fit {dt:.2f} s")
    mean, var = m.predict_batch(X[:4])
    assert np.isfinite(mean).all() and (var >= 0).all()
    assert 0.0 <= m.group_jitter(0) <= 1e-6


def test_device_fit_matches_oracle_at_config3_size():
    """The default (device) fit at n = 2048 predicts like the FP64 oracle's host fit."""
    from oracle import oracle as O
    X, Y, K = W.gp_training_set(2048, 3, seed=5)
    gd, go = G.GpModel.fit(X, Y, K), O.GP(X, Y, K)
    q = np.random.default_rng(2).uniform([-0.5, -2, -0.5, -2], [2, 2, 2, 2], size=(128, 4))
    md, vd = gd.predict_batch(q)
    mo, vo = go.predict_batch(q)
    np.testing.assert_allclose(md, mo, rtol=1e-8, atol=1e-11)
    np.testing.assert_allclose(vd, vo, rtol=0, atol=1e-10)
    for o in range(Y.shape[1]):
        assert gd.log_marginal_likelihood(o) == pytest.approx(go.lml(o), rel=1e-9)
