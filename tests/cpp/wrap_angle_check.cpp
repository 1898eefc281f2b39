// Host check: gpm::wrap_angle_fast (common.cuh) is bit-identical to gpm::wrap_angle (the
// remainder()-based wrap of core.hpp) on random, near-multiple-of-pi and half-period
// headings, zeros, huge and non-finite values. Exit code 0 on success.
#include <math.h>

#include <cstdio>
#include <cstring>
#include <random>
using std::isfinite;

#include "../../paper_2411_03289_b200/csrc/common.cuh"

int main() {
  std::mt19937_64 g(7);
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  long long bad = 0, n = 0;
  auto check = [&](double a) {
    const double x = gpm::wrap_angle_fast(a), y = gpm::wrap_angle(a);
    ++n;
    if (std::memcmp(&x, &y, 8) != 0 && !(std::isnan(x) && std::isnan(y))) {
      if (bad < 10) std::printf("mismatch a=%.17g got %.17g want %.17g\n", a, x, y);
      ++bad;
    }
  };
  const double scales[4] = {10.0, 1000.0, 1e9, 1e14};
  for (int i = 0; i < 2000000; ++i) check(u(g) * scales[i % 4]);
  for (int k = -20000; k <= 20000; ++k) {
    const double bases[2] = {k * gpm::kPi, (k + 0.5) * 2.0 * gpm::kPi};
    for (double c : bases) {
      double a = c, b = c;
      for (int j = 0; j < 6; ++j) {
        check(a);
        check(-a);
        check(b);
        a = std::nextafter(a, 1e300);
        b = std::nextafter(b, -1e300);
      }
    }
  }
  const double specials[] = {0.0, -0.0, 1e300, -1e300, INFINITY, -INFINITY, NAN, 0x1p50, -0x1p50};
  for (double a : specials) check(a);
  std::printf("%lld / %lld mismatches\n", bad, n);
  return bad != 0;
}
