"""The rollout's heading wrap (common.cuh wrap_angle_fast: rounding-trick quotient +
exact fma, no library remainder loop) is bit-identical to the remainder()-based wrap
of the reference (core.hpp wrap_angle) on random, near-tie, huge and non-finite
headings. Built for the host from the header the kernels include."""
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
