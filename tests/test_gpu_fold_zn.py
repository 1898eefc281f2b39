"""The rollout's two exponent forms against the oracle: exp(zn) folded into the combined alpha
rows (the default when the model's exponent rows are bounded, ModelDev::fold_zn) and the
unfolded q·z + qn + zn (GPMPPI_FOLD_ZN=0, the form every model outside the bound runs). The
switch is read when the model is built, hence one subprocess per form."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_ARM = r"""
import sys, dataclasses
sys.path.insert(0, {root!r})
import numpy as np
from paper_2411_03289_b200 import workloads as W
from tests.test_gpu_parity import _run_ticks
for task in ("combined", "tracking"):
    w = dataclasses.replace(W.CONFIGS["config2"], task=task, track="lane" if task != "tracking" else "circle",
                            x0=(0.0, 0.0, 0.0, 0.0, 0.0) if task != "tracking" else (2.0, 0.0, np.pi / 2, 0.0, 0.0))
    _run_ticks(w, ticks=2, samples=512)
w = dataclasses.replace(W.CONFIGS["config3"], samples=256, horizon=20)
_run_ticks(w, ticks=1, samples=256)
print("ok")
"""


@pytest.mark.parametrize("fold", ["1", "0"])
def test_rollout_exponent_forms_match_oracle(tmp_path, fold):
    script = tmp_path / "arm.py"
    script.write_text(_ARM.format(root=ROOT))
    r = subprocess.run([sys.executable, str(script)], env={**os.environ, "GPMPPI_FOLD_ZN": fold},
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout[-2000:] + r.stderr[-4000:]
