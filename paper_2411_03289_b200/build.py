"""In-tree build of the sm_100a library (nvcc, no JIT cache): lib/libgpmppi_b200.so."""
from __future__ import annotations

import os
import shutil
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "lib", "libgpmppi_b200.so")
SOURCES = ["kernels.cu", "kernels_tc.cu", "fit.cu", "capi.cpp", "hostapi.cpp"]
HEADERS = ["common.cuh", "internal.hpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def _inputs():
    files = [os.path.join(CSRC, s) for s in SOURCES + HEADERS]
    files.append(os.path.join(ROOT, "include", "gpmppi_b200.h"))
    return files


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(f) <= t for f in _inputs())


def build(force: bool = False, verbose: bool = False, variant: str = "", defines=()) -> str:
    """Build lib/libgpmppi_b200.so; `variant` + `defines` build an A/B experiment
    library lib/libgpmppi_b200_<variant>.so (selected at run time by GPMPPI_LIB)."""
    out = LIB if not variant else os.path.join(PKG, "lib", f"libgpmppi_b200_{variant}.so")
    if not variant and not force and up_to_date():
        return LIB
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    objdir = os.path.join(PKG, "lib", "obj" + (f"_{variant}" if variant else ""))
    os.makedirs(objdir, exist_ok=True)
    common = [nvcc(), "-O3", "-std=c++17", "-lineinfo", *ARCH, "-Xcompiler", "-fPIC,-O3",
              "-I", os.path.join(ROOT, "include"), "-I", CSRC, "--expt-relaxed-constexpr",
              *[f"-D{d}" for d in defines]]
    objs, procs = [], []
    for s in SOURCES:  # the translation units compile in parallel
        obj = os.path.join(objdir, os.path.splitext(s)[0] + ".o")
        cmd = common + ["-x", "cu", "-c", os.path.join(CSRC, s), "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        procs.append((s, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
        objs.append(obj)
    for s, pr in procs:
        sout, err = pr.communicate()
        if pr.returncode != 0:
            raise RuntimeError(f"nvcc failed for {s}:\n{sout}\n{err}")
        if verbose:
            print(err)
    tmp = out + ".tmp"
    cmd = [nvcc(), "-shared", *ARCH, "-o", tmp, *objs, "-cudart", "static", "-lpthread", "-ldl", "-lrt"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    import sys
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    var = next((a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--variant=")), "")
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, variant=var, defines=defs))
