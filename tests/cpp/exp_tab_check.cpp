// Host check of gpm::exp_tab (common.cuh, the tightening FP64 exp): at most 2 ulp from libm
// exp over [-700, 5] on 6M random arguments, exact 0 below -700; and of gpm::exp_tab_t (the
// rollout's, argument pre-scaled by 32/ln2): at most 2 ulp from a long-double
// exp(t·ln2/32) over the same range, exact 0 below the scaled cut.
#include <math.h>

#include <cstdio>
#include <random>
using std::isfinite;

#include "../../paper_2411_03289_b200/csrc/common.cuh"

int main() {
  double tab[32];
  for (int j = 0; j < 32; ++j) tab[j] = std::exp2(j / 32.0);
  std::mt19937_64 g(1);
  std::uniform_real_distribution<double> wide(-700.0, 5.0), gp(-40.0, 2.0), near0(-0.02, 0.02);
  double worst = 0.0, worst_x = 0.0;
  for (int i = 0; i < 6000000; ++i) {
    const double x = i % 3 == 0 ? wide(g) : i % 3 == 1 ? gp(g) : near0(g);
    const double ref = std::exp(x), got = gpm::exp_tab(x, tab);
    const double ulp = std::nextafter(ref, 1e300) - ref;
    const double e = std::fabs(got - ref) / ulp;
    if (e > worst) {
      worst = e;
      worst_x = x;
    }
  }
  const bool under = gpm::exp_tab(-700.5, tab) == 0.0 && gpm::exp_tab(-1e4, tab) == 0.0;
  std::printf("exp_tab: max %.3f ulp at x=%.17g, underflow %s\n", worst, worst_x, under ? "ok" : "BAD");
  // exp_tab_t: reference in long double from the exact scaled argument
  const long double L = logl(2.0l) / 32.0l;
  double worst_t = 0.0, worst_tx = 0.0;
  for (int i = 0; i < 6000000; ++i) {
    const double x = i % 3 == 0 ? wide(g) : i % 3 == 1 ? gp(g) : near0(g);
    const double t = x * gpm::kInvLn2x32;
    const double ref = (double)expl((long double)t * L), got = gpm::exp_tab_t(t, tab);
    const double ulp = std::nextafter(ref, 1e300) - ref;
    const double e = std::fabs(got - ref) / ulp;
    if (e > worst_t) {
      worst_t = e;
      worst_tx = t;
    }
  }
  const bool under_t = gpm::exp_tab_t(-700.5 * gpm::kInvLn2x32, tab) == 0.0 && gpm::exp_tab_t(-1e6, tab) == 0.0;
  std::printf("exp_tab_t: max %.3f ulp at t=%.17g, underflow %s\n", worst_t, worst_tx, under_t ? "ok" : "BAD");
  return worst <= 2.0 && under && worst_t <= 2.0 && under_t ? 0 : 1;
}
