"""Variance paths of the solve (FFMA, tcgen05 3xTF32, tcgen05 1xTF32, tcgen05 3xFP16 single CTA and
CTA pair) vs FP64.

var = sf2 - ||L^{-1} k*||^2 (gp.cpp:184-191) on FP32-rounded queries. Tolerances
are absolute on var (sf2 = 4e-3 for the synthetic kernel) and stated per path.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

# absolute var error bounds (sf2 = 4e-3), measured on B200 with margin:
#   FFMA ≤ 1.1e-8; 3xTF32 ≤ 1.6e-7 (fp32 tensor-core accumulation, grows with n);
#   1xTF32 ~ 8e-6 (single-pass TF32 — not a parity path, reported for the record);
#   3xFP16 (scaled operands, same 22-bit hi+lo significands as 3xTF32) shares the 3xTF32 bound,
#   single CTA (3) or CTA pair (4, tcgen05 cta_group::2: same products, other column split)
TOL = {0: 3e-8, 1: 4e-7, 2: 2e-5, 3: 4e-7, 4: 4e-7}


@pytest.mark.parametrize("n", [60, 512, 700, 2048])
@pytest.mark.parametrize("path", [0, 1, 2, 3, 4])
def test_variance_path_accuracy(n, path):
    import paper_2411_03289_b200 as G
    from paper_2411_03289_b200 import workloads as W
    X, Y, K = W.gp_training_set(n, 1, seed=n)
    m = G.GpModel.fit(X, Y, K)
    rng = np.random.default_rng(7)
    S = 1000
    q = np.column_stack([rng.uniform(-0.5, 2, S), rng.uniform(-2, 2, S),
                         rng.uniform(-0.5, 2, S), rng.uniform(-2, 2, S)])
    q32 = q.astype(np.float32).astype(np.float64)
    _, v64 = m.predict_batch(q32)
    v = m.variance_batch(q32, path)[:, 0]
    err = np.abs(v - v64[:, 0])
    print(f"n={n} path={path} max={err.max():.3e} median={np.median(err):.3e}")
    assert err.max() <= TOL[path], (n, path, err.max(), np.median(err))


@pytest.mark.parametrize("n", [1, 16, 100, 256, 272, 300, 513, 1100])
def test_pair_variance_shapes(n):
    """CTA-pair kernel: one / two 512-column passes, one or both 256-column halves, partial
    halves (n_pad not a multiple of 32), lone and partial super-tiles (S % 256 != 0)."""
    import paper_2411_03289_b200 as G
    from paper_2411_03289_b200 import workloads as W
    X, Y, K = W.gp_training_set(n, 1, seed=n + 1)
    m = G.GpModel.fit(X, Y, K)
    rng = np.random.default_rng(n)
    for S in (1, 127, 129, 255, 257, 385, 1000):
        q = np.column_stack([rng.uniform(-0.5, 2, S), rng.uniform(-2, 2, S),
                             rng.uniform(-0.5, 2, S), rng.uniform(-2, 2, S)])
        q32 = q.astype(np.float32).astype(np.float64)
        _, v64 = m.predict_batch(q32)
        v4 = m.variance_batch(q32, 4)[:, 0]
        v3 = m.variance_batch(q32, 3)[:, 0]
        assert np.abs(v4 - v64[:, 0]).max() <= TOL[4], (n, S, np.abs(v4 - v64[:, 0]).max())
        assert np.abs(v4 - v3).max() <= 1e-8, (n, S)  # same products, different summation split


def test_path3_kernel_choice_both_regimes():
    """Path 3 on a short and a long launch (3000 queries; > 16 super-tiles of 256 queries per
    CTA pair): within the path bound either way (it runs the CTA-pair kernel for n_pad > 256)."""
    import paper_2411_03289_b200 as G
    from paper_2411_03289_b200 import workloads as W
    X, Y, K = W.gp_training_set(512, 1, seed=5)
    m = G.GpModel.fit(X, Y, K)
    rng = np.random.default_rng(11)
    for S in (3000, 16 * 74 * 256 + 12345):
        q = np.column_stack([rng.uniform(-0.5, 2, S), rng.uniform(-2, 2, S),
                             rng.uniform(-0.5, 2, S), rng.uniform(-2, 2, S)])
        q32 = q.astype(np.float32).astype(np.float64)
        _, v64 = m.predict_batch(q32)
        v3 = m.variance_batch(q32, 3)[:, 0]
        v4 = m.variance_batch(q32, 4)[:, 0]
        assert np.abs(v3 - v64[:, 0]).max() <= TOL[3], S
        assert np.abs(v4 - v64[:, 0]).max() <= TOL[4], S


_SINGLE = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
import paper_2411_03289_b200 as G
from paper_2411_03289_b200 import workloads as W
TOL = {tol!r}
for n in (300, 513, 1100, 2048):
    X, Y, K = W.gp_training_set(n, 1, seed=n + 3)
    m = G.GpModel.fit(X, Y, K)
    rng = np.random.default_rng(n)
    for S in (1, 257, 3000):
        q = np.column_stack([rng.uniform(-0.5, 2, S), rng.uniform(-2, 2, S),
                             rng.uniform(-0.5, 2, S), rng.uniform(-2, 2, S)])
        q32 = q.astype(np.float32).astype(np.float64)
        _, v64 = m.predict_batch(q32)
        v3 = m.variance_batch(q32, 3)[:, 0]
        v4 = m.variance_batch(q32, 4)[:, 0]
        assert np.abs(v3 - v64[:, 0]).max() <= TOL, (n, S, np.abs(v3 - v64[:, 0]).max())
        assert np.abs(v3 - v4).max() <= 1e-8, (n, S)
print("ok")
"""


def test_single_cta_kernel_above_256_points(tmp_path):
    """The single-CTA 3xFP16 kernel (path 3 with GPMPPI_VAR2CTA=0; the default picks the CTA
    pair for n_pad > 256) against FP64 and against the pair kernel, n = 300 ... 2048. The switch
    is read once per process, hence a subprocess."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "single.py"
    script.write_text(_SINGLE.format(root=root, tol=TOL[3]))
    r = subprocess.run([sys.executable, str(script)], env={**os.environ, "GPMPPI_VAR2CTA": "0"},
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout[-2000:] + r.stderr[-3000:]
