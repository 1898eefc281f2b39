// Thin C shim over the reference's own Eigen-free RNG header
// (/root/reference/proj/include/gpmppi/rng.hpp), compiled in place by
// oracle/build_ref.sh into oracle/_ref/libref_rng.so. Used only to pin the
// oracle's RNG restatement (tests/golden/make_golden.py). The sampling loop
// restates mppi.cpp:53-62 (fill_perturbations), which itself needs Eigen.
#include <cmath>
#include <cstdint>

#include "gpmppi/rng.hpp"

extern "C" {
uint64_t ref_derive_seed(uint64_t seed, uint64_t a, uint64_t b) {
  return gpmppi::derive_seed(seed, a, b);
}
void ref_uniform_stream(uint64_t seed, int n, double* out) {
  gpmppi::RngStream r(seed);
  for (int i = 0; i < n; ++i) out[i] = r.uniform01();
}
void ref_gaussian_stream(uint64_t seed, int n, double* out) {
  gpmppi::RngStream r(seed);
  for (int i = 0; i < n; ++i) out[i] = r.gaussian();
}
void ref_sample_perturbations(int K, int T, double sv2, double sw2, uint64_t seed, uint64_t tick,
                              double* eps) {
  const double sv = std::sqrt(sv2), sw = std::sqrt(sw2);
  for (int s = 0; s < K; ++s) {
    gpmppi::RngStream rng(gpmppi::derive_seed(seed, tick, static_cast<uint64_t>(s)));
    for (int k = 0; k < T; ++k) {
      const auto [z1, z2] = rng.gaussian_pair();
      eps[(static_cast<size_t>(s) * T + k) * 2] = sv * z1;
      eps[(static_cast<size_t>(s) * T + k) * 2 + 1] = sw * z2;
    }
  }
}
}
