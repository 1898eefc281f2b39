"""The reference-shaped C++ header (include/gpmppi/planner.hpp) compiles and links
against the in-tree library; on CPU the first compute call raises std::runtime_error
(CUDA error, no fallback); on a B200 the three plan_step overloads run."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2411_03289_b200", "lib")


def _build(tmp_path, name="example_planner"):
    exe = str(tmp_path / name)
    cmd = ["g++", "-std=c++17", "-O1", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", name + ".cpp"), "-L", LIBDIR,
           "-lgpmppi_b200", f"-Wl,-rpath,{LIBDIR}", "-o", exe]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
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


def test_eigen_typed_callers_compile_and_run_host_calls(tmp_path):
    """Caller code passing Eigen-shaped types (a minimal stand-in with rows(), cols(), v(i),
    m(i, j)) compiles against planner.hpp; its host-only calls run without a GPU."""
    exe = _build(tmp_path, "eigen_stub_caller")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=60)
    first = r.stdout.splitlines()[0]
    assert first.startswith("host sigma=(0.300, 0.500) circle=1 lane_wp=2 x0=(2.0, 1.5708) ls2=0.8 nx_v=0.200 J33=0.90"), r.stdout
    if not _has_gpu():
        assert r.returncode == 2 and "runtime_error" in r.stdout, r.stdout + r.stderr


@pytest.mark.gpu
def test_eigen_typed_callers_on_gpu(tmp_path):
    exe = _build(tmp_path, "eigen_stub_caller")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    dev = r.stdout.splitlines()[1]
    assert dev.startswith("device pred=") and "states=13" in dev and "radii=12" in dev
