"""Device math helpers checked on the host, built from the header the kernels include
(common.cuh): the heading wrap (wrap_angle_fast: rounding-trick quotient + exact fma)
is bit-identical to the reference's remainder()-based wrap (core.hpp wrap_angle) on
random, near-tie, huge and non-finite headings; the table-driven FP64 exp of the GP
kernel row (exp_tab) stays within 2 ulp of libm."""
import os
import shutil
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.skipif(shutil.which("g++") is None, reason="g++ not available")
def test_wrap_angle_fast_bit_identical(tmp_path):
    exe = str(tmp_path / "wac")
    subprocess.run(["g++", "-O2", "-ffp-contract=off", "-std=c++17", "-o", exe,
                    os.path.join(HERE, "cpp", "wrap_angle_check.cpp")], check=True)
    r = subprocess.run([exe], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.strip().startswith("0 /")


@pytest.mark.skipif(shutil.which("g++") is None, reason="g++ not available")
def test_exp_tab_within_two_ulp(tmp_path):
    """The table-driven FP64 exp of the GP kernel row (common.cuh exp_tab) vs libm."""
    exe = str(tmp_path / "etc")
    subprocess.run(["g++", "-O2", "-ffp-contract=off", "-std=c++17", "-o", exe,
                    os.path.join(HERE, "cpp", "exp_tab_check.cpp")], check=True)
    r = subprocess.run([exe], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
