#!/usr/bin/env bash
# Compiles the only Eigen-free piece of the reference (include/gpmppi/rng.hpp)
# from the read-only tree into oracle/_ref/ (git-ignored). The rest of the
# reference needs Eigen3/doctest/CLI11/json.hpp, which are absent: unbuildable.
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
ref="${GPMPPI_REFERENCE:-/root/reference}/proj/include"
if [ ! -f "$ref/gpmppi/rng.hpp" ]; then
  echo "reference not present; skipping oracle/_ref build" >&2
  exit 0
fi
mkdir -p "$here/_ref"
g++ -std=c++20 -O2 -fPIC -shared -I"$ref" "$here/ref_rng_shim.cpp" -o "$here/_ref/libref_rng.so"
echo "built $here/_ref/libref_rng.so"
