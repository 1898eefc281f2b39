"""The pipelined single-robot tightening pass (publisher / stager / recursion warps in the mean
kernel, the variance grid released step by step) against the sequential three-kernel pass
(GPMPPI_TIGHTEN_SEQUENTIAL=1): the same arithmetic in the same orders, so the lane radii, the
obstacle margins, the horizon covariances and the infeasibility flag must be bit-identical.
The setting is read once per process, hence one subprocess per arm."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_ARM = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
import paper_2411_03289_b200 as G
from paper_2411_03289_b200 import workloads as W
from tests.helpers import build_pair
import dataclasses
name, _, horizon = sys.argv[1].partition(":")
w = W.CONFIGS[name]
if horizon:
    w = dataclasses.replace(w, horizon=int(horizon))
_, pd, _, td, _ = build_pair(w, samples=int(sys.argv[3]))
x = np.array(w.x0)
out = {{}}
for t in range(3):
    d = G.StepDiagnostics()
    cmd = pd.plan_step(x, td, d)
    out[f"radii{{t}}"] = pd.lane_radii()
    out[f"cov{{t}}"] = pd.horizon_covariances()
    out[f"inf{{t}}"] = np.array([int(d.tightening_infeasible)])
    if w.task in ("avoidance", "combined"):
        out[f"marg{{t}}"] = pd.obstacle_margins()
    x = x + np.array([0.01, 0.0, 0.002, 0.0, 0.0])
np.savez(sys.argv[2], **out)
"""


@pytest.mark.parametrize("cfg,samples", [("config2", 1024), ("config3", 512), ("config1", 512),
                                         ("config2:1", 256), ("config2:2", 256), ("config2:33", 256),
                                         ("config2:97", 256)])
def test_pipelined_tightening_matches_sequential(tmp_path, cfg, samples):
    script = tmp_path / "arm.py"
    script.write_text(_ARM.format(root=ROOT))
    res = {}
    for seq in ("0", "1"):
        f = str(tmp_path / f"{cfg.replace(':', '_')}_{seq}.npz")
        env = {**os.environ, "GPMPPI_TIGHTEN_SEQUENTIAL": seq}
        r = subprocess.run([sys.executable, str(script), cfg, f, str(samples)], env=env, capture_output=True,
                           text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-3000:]
        res[seq] = np.load(f)
    a, b = res["0"], res["1"]
    assert sorted(a.files) == sorted(b.files)
    for k in a.files:
        np.testing.assert_array_equal(a[k], b[k], err_msg=f"{cfg}: {k}")


@pytest.mark.parametrize("serialise", [{"GPMPPI_NO_PDL": "1"}, {"GPMPPI_NO_GRAPH": "1", "GPMPPI_DEBUG_SYNC": "1"}])
def test_pipelined_tightening_survives_serialised_kernels(tmp_path, serialise):
    """The pipelined pass only waits on kernels launched before the waiter, so it completes (with
    the same results) when the kernels cannot overlap: no programmatic dependent launch, or a
    synchronisation after every launch (as under a serialising profiler)."""
    script = tmp_path / "arm.py"
    script.write_text(_ARM.format(root=ROOT))
    res = {}
    for tag, extra in (("overlap", {}), ("serial", serialise)):
        f = str(tmp_path / f"{tag}.npz")
        env = {**os.environ, "GPMPPI_TIGHTEN_SEQUENTIAL": "0", **extra}
        r = subprocess.run([sys.executable, str(script), "config2", f, "512"], env=env, capture_output=True,
                           text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-3000:]
        res[tag] = np.load(f)
    for k in res["overlap"].files:
        np.testing.assert_array_equal(res["overlap"][k], res["serial"][k], err_msg=k)
