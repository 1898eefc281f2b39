// hostapi.cpp — the reference's scalar free functions behind the C ABI (host C++).
//
// These are the per-call helpers the reference exports next to the planner
// (bindings/module.cpp:40-181): dynamics steps and their Jacobian, the kernel,
// the terrain combine, the simplex projection, the quantiles and the two
// tightening rules. They are a few dozen FLOPs each and run on the host, as in
// the reference; the arithmetic is the same __host__ __device__ code the planner's
// kernels run (common.cuh), so a host call and the device tick agree bit for bit
// on dynamics. Argument checks and messages follow the reference's throws.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include "gpmppi_b200.h"
#include "internal.hpp"

namespace gpm_host {
int set_error(int code, const std::string& msg);  // capi.cpp
}

namespace {

bool finite_n(const double* v, int n) {
  for (int i = 0; i < n; ++i)
    if (!std::isfinite(v[i])) return false;
  return true;
}
int bad(const std::string& m) { return gpm_host::set_error(GPMPPI_INVALID_ARGUMENT, m); }
// dynamics.cpp:11-15 check_finite
bool state_control_finite(const double* s, const double* u) { return finite_n(s, 5) && finite_n(u, 2); }
// dynamics.cpp:18-25 NominalParams::validate
const char* nominal_invalid(const gpmppi_nominal* p) {
  if (!p) return "NominalParams: null";
  if (!(p->tau_v > 0.0) || !(p->tau_omega > 0.0)) return "NominalParams: time constants must be positive";
  if (!(p->dt > 0.0) || p->dt >= std::min(p->tau_v, p->tau_omega))
    return "NominalParams: require 0 < dt < min(tau_v, tau_omega)";
  return nullptr;
}
double lambda_max_2x2(const double* m) {  // uncertainty.cpp:62-66
  const double half_tr = 0.5 * (m[0] + m[3]);
  const double det_disc = 0.25 * (m[0] - m[3]) * (m[0] - m[3]) + m[1] * m[2];
  return half_tr + std::sqrt(std::max(det_disc, 0.0));
}
double acklam(double p) {  // uncertainty.cpp:19-52
  static const double a[] = {-3.969683028665376e+01, 2.209460984245205e+02, -2.759285104469687e+02,
                             1.383577518672690e+02,  -3.066479806614716e+01, 2.506628277459239e+00};
  static const double b[] = {-5.447609879822406e+01, 1.615858368580409e+02, -1.556989798598866e+02,
                             6.680131188771972e+01,  -1.328068155288572e+01};
  static const double c[] = {-7.784894002430293e-03, -3.223964580411365e-01, -2.400758277161838e+00,
                             -2.549732539343734e+00, 4.374664141464968e+00,  2.938163982698783e+00};
  static const double d[] = {7.784695709041462e-03, 3.224671290700398e-01, 2.445134137142996e+00,
                             3.754408661907416e+00};
  const double plow = 0.02425;
  if (p < plow) {
    const double q = std::sqrt(-2.0 * std::log(p));
    return (((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
           ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1.0);
  }
  if (p > 1.0 - plow) {
    const double q = std::sqrt(-2.0 * std::log(1.0 - p));
    return -(((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
           ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1.0);
  }
  const double q = p - 0.5, r = q * q;
  return (((((a[0] * r + a[1]) * r + a[2]) * r + a[3]) * r + a[4]) * r + a[5]) * q /
         (((((b[0] * r + b[1]) * r + b[2]) * r + b[3]) * r + b[4]) * r + 1.0);
}
double ncdf(double x) { return 0.5 * std::erfc(-x * 0.70710678118654752440); }  // uncertainty.cpp:15
bool quantile(double p, double* out) {  // uncertainty.cpp:54-60
  if (!(p > 0.0) || !(p < 1.0)) return false;
  double x = acklam(p);
  const double pdf = std::exp(-0.5 * x * x) / std::sqrt(2.0 * gpm::kPi);
  if (pdf > 1e-300) x -= (ncdf(x) - p) / pdf;
  *out = x;
  return true;
}
bool on_simplex(const double* w, int m, double tol) {  // core.hpp:107-111
  if (m <= 0) return false;
  double s = 0.0;
  for (int i = 0; i < m; ++i) s += w[i];
  if (std::fabs(s - 1.0) > tol) return false;
  for (int i = 0; i < m; ++i)
    if (!(w[i] >= -tol) || !(w[i] <= 1.0 + tol)) return false;
  return true;
}

}  // namespace

extern "C" {

double gpmppi_wrap_angle(double a) { return gpm::wrap_angle(a); }  // core.hpp:18-27

int gpmppi_step_nominal(const double s[5], const double u[2], const gpmppi_nominal* p, double out[5]) {
  if (const char* e = nominal_invalid(p)) return bad(e);
  if (!state_control_finite(s, u)) return bad("step_nominal: non-finite input");
  double s0, c0;
  gpm::sincos_d(s[2], &s0, &c0);
  gpm::step_nominal(s, u, gpm::NominalDev{p->tau_v, p->tau_omega, p->dt}, out, s0, c0);
  return GPMPPI_OK;
}

int gpmppi_step_kinematic_unicycle(const double s[5], const double u[2], double dt, double out[5]) {
  if (!state_control_finite(s, u)) return bad("step_kinematic_unicycle: non-finite input");
  gpm::step_kinematic(s, u, dt, out);
  return GPMPPI_OK;
}

int gpmppi_step_edd5(const double s[5], const double u[2], const gpmppi_edd5* p, double track_width, double dt,
                     double out[5]) {
  if (!p) return bad("step_edd5: null parameters");
  if (!state_control_finite(s, u)) return bad("step_edd5: non-finite input");
  if (!(track_width > 0.0)) return bad("step_edd5: track_width must be positive");
  if (p->y_icr_r - p->y_icr_l <= 1e-6) return bad("step_edd5: degenerate ICR span (y_icr_r - y_icr_l <= 1e-6)");
  gpm::step_edd5(s, u, gpm::Edd5Dev{p->alpha_l, p->alpha_r, p->x_icr, p->y_icr_l, p->y_icr_r, track_width}, dt, out);
  return GPMPPI_OK;
}

int gpmppi_jacobian_nominal(const double s[5], const double u[2], const gpmppi_nominal* p, double J[25]) {
  if (const char* e = nominal_invalid(p)) return bad(e);
  if (!state_control_finite(s, u)) return bad("jacobian_nominal: non-finite input");
  gpm::jacobian_nominal(s, gpm::NominalDev{p->tau_v, p->tau_omega, p->dt}, J);
  return GPMPPI_OK;
}

int gpmppi_body_frame_displacement(const double from[5], const double to[5], double out[2]) {  // core.hpp:117-126
  if (!finite_n(from, 5) || !finite_n(to, 5)) return bad("body_frame_displacement: non-finite state");
  const double dx = to[0] - from[0], dy = to[1] - from[1];
  const double c = std::cos(from[2]), s = std::sin(from[2]);
  out[0] = c * dx + s * dy;
  out[1] = -s * dx + c * dy;
  return GPMPPI_OK;
}

int gpmppi_kernel_eval(const double a[4], const double b[4], const double kernel6[6], double* out) {  // gp.cpp:53-60
  bool ok = kernel6[0] > 0.0 && kernel6[5] > 0.0;
  for (int d = 0; d < 4; ++d) ok = ok && kernel6[1 + d] > 0.0;
  if (!ok) return bad("KernelParams: all parameters must be strictly positive");
  if (!finite_n(a, 4) || !finite_n(b, 4)) return bad("kernel_eval: non-finite input");
  double sq = 0.0;
  for (int d = 0; d < 4; ++d) {
    const double t = (a[d] - b[d]) / kernel6[1 + d];
    sq += t * t;
  }
  *out = kernel6[0] * std::exp(-0.5 * sq);
  return GPMPPI_OK;
}

int gpmppi_ensemble_combine(const double* means, const double* var_diags, const double* w, int m, double mean[2],
                            double cov[4]) {  // gp.cpp:368-389 (means, var_diags: m x 2 row-major)
  if (m < 1 || !means || !var_diags || !w) return bad("ensemble_combine: size mismatch");
  if (!on_simplex(w, m, 1e-6)) return bad("ensemble_combine: weights off the simplex beyond 1e-6");
  double m0 = 0.0, m1 = 0.0, vv = 0.0, vw = 0.0;
  for (int i = 0; i < m; ++i) {
    m0 += w[i] * means[2 * i];
    m1 += w[i] * means[2 * i + 1];
    vv += w[i] * w[i] * var_diags[2 * i];
    vw += w[i] * w[i] * var_diags[2 * i + 1];
  }
  mean[0] = m0;
  mean[1] = m1;
  cov[0] = vv;
  cov[1] = cov[2] = 0.0;
  cov[3] = vw;
  return GPMPPI_OK;
}

int gpmppi_project_simplex(const double* z, int m, double* out) {  // terrain.cpp:72-92
  if (m < 1 || !z || !finite_n(z, m)) return bad("project_simplex: need a finite non-empty vector");
  std::vector<double> u(z, z + m);
  std::sort(u.begin(), u.end(), std::greater<double>());
  double cumsum = 0.0, tau = 0.0;
  for (int i = 0; i < m; ++i) {
    cumsum += u[i];
    const double t = (cumsum - 1.0) / (double)(i + 1);
    if (u[i] - t > 0.0) tau = t;
  }
  for (int i = 0; i < m; ++i) out[i] = std::max(z[i] - tau, 0.0);
  return GPMPPI_OK;
}

int gpmppi_chi2_quantile_2dof(double p, double* out) {  // uncertainty.cpp:8-13
  if (!(p >= 0.0) || p >= 1.0) return bad("chi2_quantile_2dof: p must lie in [0, 1)");
  *out = -2.0 * std::log1p(-p);
  return GPMPPI_OK;
}

int gpmppi_normal_quantile(double p, double* out) {
  if (!quantile(p, out)) return bad("normal_quantile: p must lie in (0, 1)");
  return GPMPPI_OK;
}

double gpmppi_normal_cdf(double x) { return ncdf(x); }

int gpmppi_tighten_lane_radius(double r, const double cov_xy[4], double p_x, double* out) {  // uncertainty.cpp:90-96
  if (!(p_x > 0.5) || !(p_x < 1.0)) return bad("QuantileTables: p_x must lie in (0.5, 1)");
  if (!(r > 0.0)) return bad("tighten_lane_radius: r must be positive");
  const double chi2 = -2.0 * std::log1p(-p_x);
  *out = r - std::sqrt(chi2 * std::max(lambda_max_2x2(cov_xy), 0.0));
  return GPMPPI_OK;
}

int gpmppi_tighten_obstacle_distance(const double robot_xy[2], const double center[2], double radius,
                                     const double cov_xy[4], double p_x, double* d_bar, double normal[2],
                                     int* degenerate, double* d) {  // uncertainty.cpp:98-116
  if (!(p_x > 0.5) || !(p_x < 1.0)) return bad("QuantileTables: p_x must lie in (0.5, 1)");
  double z = 0.0;
  quantile(p_x, &z);
  const double dx = robot_xy[0] - center[0], dy = robot_xy[1] - center[1];
  const double dist = std::sqrt(dx * dx + dy * dy);
  double n0, n1, dd;
  int deg = 0;
  if (dist < 1e-12) {
    deg = 1;
    n0 = 1.0;
    n1 = 0.0;
    dd = -radius;
  } else {
    n0 = dx / dist;
    n1 = dy / dist;
    dd = dist - radius;
  }
  // n . (C n), C row-major
  const double cn0 = cov_xy[0] * n0 + cov_xy[1] * n1, cn1 = cov_xy[2] * n0 + cov_xy[3] * n1;
  const double dir_var = std::max(n0 * cn0 + n1 * cn1, 0.0);
  if (d_bar) *d_bar = dd - z * std::sqrt(dir_var);
  if (normal) {
    normal[0] = n0;
    normal[1] = n1;
  }
  if (degenerate) *degenerate = deg;
  if (d) *d = dd;
  return GPMPPI_OK;
}

}  // extern "C"
