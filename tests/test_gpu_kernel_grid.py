"""select_kernel_grid (gp.cpp:274-366) on the device vs the CPU restatement (oracle).

Both sweep the reference's coarse 5x7x5 grid and one 5x7x5 refinement with the
first-strictly-greater argmax; the device factors every cell (FP64 Cholesky per CTA,
csrc/fit.cu) and the oracle uses numpy's LAPACK Cholesky, so the chosen cell must be the
same and the winning LML agree to rounding (rtol 1e-9).
"""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _check(X, Y):
    from paper_2411_03289_b200 import harness as H
    k = H.select_kernel_grid(X, Y)
    sv, ls, nv, lml = O.select_kernel_grid(X, Y)
    assert k.signal_var == pytest.approx(sv, rel=1e-12)
    np.testing.assert_allclose(k.lengthscales, ls, rtol=1e-12)
    assert k.noise_var == pytest.approx(nv, rel=1e-12)
    return k, lml


@pytest.mark.parametrize("n,m,seed", [(2, 1, 0), (60, 2, 4), (137, 6, 1), (300, 6, 2)])
def test_grid_matches_cpu_restatement(n, m, seed):
    rng = np.random.default_rng(seed)
    X = np.column_stack([rng.uniform(-0.5, 2.0, n), rng.uniform(-2, 2, n), rng.uniform(-0.5, 2.0, n),
                         rng.uniform(-2, 2, n)])
    Y = np.column_stack([0.02 * np.sin(X[:, 0] + j) + 0.01 * X[:, 2] - 0.003 * j * X[:, 3] for j in range(m)])
    Y += 1e-3 * rng.normal(size=Y.shape)
    _check(X, Y)


def test_grid_on_harness_training_data():
    """The closed loop's training set (harness.cpp:190-243): 3 terrains, 300 shared inputs."""
    from paper_2411_03289_b200 import harness as H
    import paper_2411_03289_b200 as G
    cfg = H.ExperimentConfig()
    m = len(cfg.terrains)
    per = [H.generate_training_data(cfg.terrains[i], cfg.nominal, cfg.mppi.bounds, 300,
                                    H.RngStream(H.derive_seed(0, 100 + i))) for i in range(m)]
    X = np.stack([per[r % m][0][r] for r in range(300)])
    Y = np.column_stack([per[r % m][1][:, c] for r in range(1) for c in range(2)] * m)
    k, _ = _check(X, Y[:, : 2 * m])
    gp = G.GpModel.fit(X, Y[:, : 2 * m], [k] * (2 * m))
    assert np.isfinite(gp.log_marginal_likelihood(0))


def test_grid_errors():
    from paper_2411_03289_b200 import harness as H
    with pytest.raises(ValueError):
        H.select_kernel_grid(np.zeros((1, 4)), np.zeros((1, 1)))
