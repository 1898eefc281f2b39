"""On-disk model formats: GPMPPIG1 (gp.cpp:223-272) inside
GPMPPIM1 (harness.cpp:249-284). The committed fixtures follow the reference
writers byte for byte (tests/golden/make_models_golden.py); the device library
must read them and write back identical bytes."""
import os
import struct

import numpy as np
import pytest

from tests.golden.make_models_golden import models_bytes, small_case

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_fixture_layout_matches_reference_writers():
    X, Y, kernels, edd5, nominal = small_case()
    raw = open(os.path.join(GOLD, "models_small.gpm"), "rb").read()
    assert raw == models_bytes(X, Y, kernels, edd5, nominal)
    assert raw[:8] == b"GPMPPIM1" and raw[8 + 64 + 1:8 + 64 + 9] == b"GPMPPIG1"
    assert struct.unpack("<5d", raw[8:48]) == edd5 and struct.unpack("<3d", raw[48:72]) == nominal
    n, m = struct.unpack("<qq", raw[81:97])
    assert (n, m) == (7, 4) and len(raw) == 97 + 8 * (4 * n + n * m + 6 * m)
    col0 = np.frombuffer(raw[97:97 + 8 * n], dtype="<f8")
    np.testing.assert_array_equal(col0, X[:, 0])  # column-major inputs
    nogp = open(os.path.join(GOLD, "models_nogp.gpm"), "rb").read()
    assert len(nogp) == 73 and nogp[72] == 0


@pytest.mark.gpu
def test_models_file_round_trip_bit_exact(tmp_path):
    import paper_2411_03289_b200 as G
    X, Y, kernels, edd5, nominal = small_case()
    m = G.load_models(os.path.join(GOLD, "models_small.gpm"))
    assert m.has_gp and m.gp.n_points == 7 and m.gp.n_outputs == 4
    assert (m.edd5.alpha_l, m.edd5.alpha_r, m.edd5.x_icr, m.edd5.y_icr_l, m.edd5.y_icr_r) == edd5
    assert (m.nominal.tau_v, m.nominal.tau_omega, m.nominal.dt) == nominal
    Xb, Yb = m.gp.training_data()
    np.testing.assert_array_equal(Xb, X)
    np.testing.assert_array_equal(Yb, Y)
    out = str(tmp_path / "rt.gpm")
    G.save_models(out, m)
    assert open(out, "rb").read() == open(os.path.join(GOLD, "models_small.gpm"), "rb").read()
    ref = G.GpModel.fit(X, Y, kernels)  # the loaded model predicts like a fresh fit
    q = np.array([[0.4, 0.2, 1.1, -0.3], [1.5, -1.0, 0.0, 0.7]])
    np.testing.assert_array_equal(m.gp.predict_batch(q)[0], ref.predict_batch(q)[0])
    e = G.load_models(os.path.join(GOLD, "models_nogp.gpm"))
    assert not e.has_gp and e.gp is None
    G.save_models(out, e)
    assert open(out, "rb").read() == open(os.path.join(GOLD, "models_nogp.gpm"), "rb").read()
    bad = tmp_path / "bad.gpm"
    bad.write_bytes(b"GPMPPIX1" + b"\0" * 80)
    with pytest.raises(RuntimeError):
        G.load_models(str(bad))
    bad.write_bytes(b"GPMPPIM1" + b"\0" * 10)
    with pytest.raises(RuntimeError):
        G.load_models(str(bad))
