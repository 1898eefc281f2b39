"""The reference-shaped C++ header (include/gpmppi/planner.hpp) compiles and links
against the in-tree library; on CPU the first compute call raises std::runtime_error
(CUDA error, no fallback); on a B200 the three plan_step overloads run."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2411_03289_b200", "lib")


def _build(tmp_path):
    exe = str(tmp_path / "example_planner")
    cmd = ["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", "example_planner.cpp"), "-L", LIBDIR,
           "-lgpmppi_b200", f"-Wl,-rpath,{LIBDIR}", "-o", exe]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def test_header_compiles_links_and_raises_without_gpu(tmp_path):
    exe = _build(tmp_path)
    if _has_gpu():
        pytest.skip("GPU present: covered by the gpu test")
    r = subprocess.run([exe], capture_output=True, text=True)
    assert r.returncode == 2 and "runtime_error" in r.stdout, r.stdout + r.stderr


@pytest.mark.gpu
def test_header_plan_step_on_gpu(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    lines = r.stdout.strip().splitlines()
    assert lines[0].startswith("tracking") and lines[2].startswith("combined")
    assert "radii=20" in lines[2]
    assert lines[3].startswith("free") and "w0=0.731058578630" in lines[3] and "states=21" in lines[3]
    assert "eps=512x20" in lines[3] and lines[4].startswith("batch") and "robots=3" in lines[4]
