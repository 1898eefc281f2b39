"""Writes tests/golden/models_small.gpm: a GPMPPIM1 models file laid out exactly as
the reference writers lay it out (harness.cpp:249-262 save_models around
gp.cpp:230-242 GpModel::save). The reference cannot be built here (Eigen is absent,
SURVEY §8(c)), so the bytes are produced by this restatement of its writers:
  'GPMPPIM1' | edd5 5xf64 | nominal 3xf64 | has_gp u8 |
  'GPMPPIG1' | n i64 | m i64 | inputs n x 4 col-major f64 | outputs n x m col-major f64 |
  per output: signal_var, lengthscales[4], noise_var (f64)
Run: python tests/golden/make_models_golden.py
"""
import os
import struct

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def models_bytes(X, Y, kernels, edd5, nominal, has_gp=True):
    b = b"GPMPPIM1" + struct.pack("<5d", *edd5) + struct.pack("<3d", *nominal) + bytes([1 if has_gp else 0])
    if has_gp:
        n, m = X.shape[0], Y.shape[1]
        b += b"GPMPPIG1" + struct.pack("<qq", n, m)
        b += np.asfortranarray(X).tobytes(order="F") + np.asfortranarray(Y).tobytes(order="F")
        for k in kernels:
            b += struct.pack("<6d", *k)
    return b


def small_case():
    rng = np.random.default_rng(2024)
    n = 7
    X = np.column_stack([rng.uniform(-0.5, 2, n), rng.uniform(-2, 2, n), rng.uniform(-0.5, 2, n),
                         rng.uniform(-2, 2, n)])
    Y = np.column_stack([0.02 * np.sin(X[:, 0]) + 0.01 * X[:, 2], -0.015 * X[:, 3],
                         0.02 * np.sin(X[:, 0] + 1) + 0.01 * X[:, 2], -0.015 * X[:, 3] + 0.005])
    kernels = [(4e-3, 0.8, 1.2, 0.8, 1.2, 1e-4)] * 4
    edd5 = (0.93, 0.97, 0.015, -0.21, 0.19)
    nominal = (0.45, 0.3, 0.05)
    return X, Y, kernels, edd5, nominal


if __name__ == "__main__":
    X, Y, kernels, edd5, nominal = small_case()
    with open(os.path.join(HERE, "models_small.gpm"), "wb") as f:
        f.write(models_bytes(X, Y, kernels, edd5, nominal))
    with open(os.path.join(HERE, "models_nogp.gpm"), "wb") as f:
        f.write(models_bytes(None, None, None, edd5, nominal, has_gp=False))
    print("wrote models_small.gpm, models_nogp.gpm")
