// common.cuh — device-side restatement of the per-sample math of the GP-MPPI
// solve (FP64 state path) plus the Philox sampler and the reduction tuple.
// Each function cites the reference (/root/reference/proj) lines it follows.
#pragma once

#include <cstdint>
#include <cmath>
#include <cstring>

#if defined(__CUDACC__)
#define GPM_HD __host__ __device__ __forceinline__
#define GPM_D __device__ __forceinline__
#else
#define GPM_HD inline
#define GPM_D inline
#endif

namespace gpm {

constexpr double kPi = 3.14159265358979323846;  // core.hpp:14
constexpr int kMaxWaypoints = 64;
constexpr int kMaxObstacles = 64;
constexpr int kMaxTerrains = 16;
constexpr int kMaxGroups = 4;
#ifndef GPM_MAX_OUT_PER_GROUP
#define GPM_MAX_OUT_PER_GROUP (2 * kMaxTerrains)
#endif
constexpr int kMaxOutPerGroup = GPM_MAX_OUT_PER_GROUP;  // one shared kernel over every terrain (harness.cpp:242-244)
constexpr int kOutChunk = 8;  // outputs whose alpha loads are kept in flight together

enum { TASK_TRACKING = 0, TASK_AVOIDANCE = 1, TASK_COMBINED = 2 };
enum { MODEL_GP = 0, MODEL_EDD5 = 1, MODEL_UNICYCLE = 2, MODEL_NOMINAL = 3 };

// Per-tick task view (mppi.hpp:42-52), resident in device memory.
struct TaskDev {
  int kind;
  int is_circle;
  int n_wp;
  int closed;
  int n_obs;
  int pad_;
  double cx, cy, radius, half_width;
  double v_desired;
  double tw[5];  // variance, deviation, slip, safety, speed   (costs.hpp:34-40)
  double aw[4];  // variance, obstacle, stage, terminal        (costs.hpp:44-50)
  double goal[3];
  double high_cost;
  double wp[kMaxWaypoints][2];
  double obs[kMaxObstacles][3];
};

struct NominalDev {
  double tau_v, tau_omega, dt;
};
struct Edd5Dev {
  double alpha_l, alpha_r, x_icr, y_icr_l, y_icr_r, track_width;
};

// core.hpp:18-27 — remainder() is exact in IEEE arithmetic, so this matches libm bit for bit.
// 32-bit halves of a double (device intrinsics; memcpy on the host)
GPM_HD int dbl_lo(double d) {
#if defined(__CUDA_ARCH__)
  return __double2loint(d);
#else
  uint64_t u;
  std::memcpy(&u, &d, 8);
  return (int)(uint32_t)u;
#endif
}
GPM_HD int dbl_hi(double d) {
#if defined(__CUDA_ARCH__)
  return __double2hiint(d);
#else
  uint64_t u;
  std::memcpy(&u, &d, 8);
  return (int)(uint32_t)(u >> 32);
#endif
}
GPM_HD double dbl_from(int hi, int lo) {
#if defined(__CUDA_ARCH__)
  return __hiloint2double(hi, lo);
#else
  const uint64_t u = ((uint64_t)(uint32_t)hi << 32) | (uint32_t)lo;
  double d;
  std::memcpy(&d, &u, 8);
  return d;
#endif
}

// FP64 exp for the GP kernel row: exp(x) = 2^(n/32)·e^r, n = rint(32x/ln2),
// |r| <= ln2/64, e^r - 1 = r + r^2·q(r) with q a degree-3 minimax fit of
// ((e^r-1)/r - 1)/r (Remez, relative error 1.3e-14 on q's range, i.e. <= 1.5e-16
// on the result), and a 32-entry 2^(j/32) table in shared memory. 11 FP64 ops
// instead of ~22 for libm's exp; max 2 ulp from libm over [-700, 5] (20M-point
// host sweep); arguments below -700 flush to 0 (k* < 1e-304).
constexpr double kInvLn2x32 = 0x1.71547652b82fep+5;
constexpr double kLn2d32Hi = 0x1.62e42fee00000p-6;  // 32 significant bits: n·hi exact for |n| < 2^21
constexpr double kLn2d32Lo = 0x1.a39ef35793c76p-38;
GPM_HD double exp_tab(double x, const double* tab) {
  const double magic = 6755399441055744.0;  // 1.5·2^52: round-to-nearest integer trick
  const double t = fma(x, kInvLn2x32, magic);
  const int n = dbl_lo(t);
  const double nd = t - magic;
  double r = fma(nd, -kLn2d32Hi, x);
  r = fma(nd, -kLn2d32Lo, r);
  double q = fma(0x1.1111688fec18cp-7, r, 0x1.5555c2a9cb753p-5);
  q = fma(q, r, 0x1.5555555541cedp-3);
  q = fma(q, r, 0x1.ffffffffe5bc7p-2);
  const double p = fma(r * r, q, r);  // e^r - 1
  const double tj = tab[n & 31];
  const double res = fma(tj, p, tj);
  const double scaled = dbl_from(dbl_hi(res) + ((n >> 5) << 20), dbl_lo(res));
  return x < -700.0 ? 0.0 : scaled;
}

// exp_tab of an argument already scaled by 32/ln2 (t = 32x/ln2; the rollout folds the scale
// into its staged kernel points): n = rint(t), s = t - n is exact (Sterbenz), and
// e^(s·ln2/32) - 1 is exp_tab's polynomial with the scale folded into its coefficients
// (b_i = c_i·(ln2/32)^i, Horner in s). 10 FP64 ops instead of 11: the reduction is one
// DADD instead of two DFMAs. Within 2 ulp of exp(t·ln2/32) (tests/cpp/exp_tab_check.cpp);
// t below -700·32/ln2 flushes to 0, as exp_tab.
constexpr double kLn2d32 = 0x1.62e42fefa39efp-6;
constexpr double kExpTB1 = kLn2d32;
constexpr double kExpTB2 = 0x1.ffffffffe5bc7p-2 * kLn2d32 * kLn2d32;
constexpr double kExpTB3 = 0x1.5555555541cedp-3 * kLn2d32 * kLn2d32 * kLn2d32;
constexpr double kExpTB4 = 0x1.5555c2a9cb753p-5 * kLn2d32 * kLn2d32 * kLn2d32 * kLn2d32;
constexpr double kExpTB5 = 0x1.1111688fec18cp-7 * kLn2d32 * kLn2d32 * kLn2d32 * kLn2d32 * kLn2d32;
constexpr double kExpTMin = -700.0 * kInvLn2x32;
GPM_HD double exp_tab_t(double t, const double* tab) {
  const double magic = 6755399441055744.0;
  const double tt = t + magic;
  const int n = dbl_lo(tt);
  const double s = t - (tt - magic);
  double u = fma(kExpTB5, s, kExpTB4);
  u = fma(u, s, kExpTB3);
  u = fma(u, s, kExpTB2);
  u = fma(u, s, kExpTB1);
  const double p = u * s;  // e^(s·ln2/32) - 1
  const double tj = tab[n & 31];
  const double res = fma(tj, p, tj);
  const double scaled = dbl_from(dbl_hi(res) + ((n >> 5) << 20), dbl_lo(res));
  return t < kExpTMin ? 0.0 : scaled;
}

GPM_HD double wrap_angle(double a) {
  double r = remainder(a, 2.0 * kPi);
  if (r <= -kPi) r += 2.0 * kPi;
  return r;
}
// wrap_angle without the library remainder (~200-cycle dependent chain per call; the
// rollout's heading recursion is serial in k): n = rint(a / 2π) by the 1.5·2^52
// rounding trick, r = fma(-n, 2π, a) -- exact, since an IEEE remainder is
// representable -- and one select each way when n was off by one. Bit-identical to
// wrap_angle, including the sign of a zero result (tests/test_wrap_angle.py).
GPM_HD double wrap_angle_fast(double a) {
  const double P = 2.0 * kPi, magic = 6755399441055744.0;
  if (!(fabs(a) < 0x1p50)) return wrap_angle(a);  // huge or non-finite
  const double n = fma(a, 1.0 / (2.0 * kPi), magic) - magic;
  double r = fma(-n, P, a);
  r = r > kPi ? r - P : r;  // Sterbenz: exact
  r = r < -kPi ? r + P : r;
  r = r == 0.0 ? copysign(0.0, a) : r;
  return r <= -kPi ? r + P : r;
}

// dynamics.cpp:39-57 (sin/cos of theta passed in: s0 = sin(theta), c0 = cos(theta)).
GPM_HD void arc_advance(double& x, double& y, double& th, double vx, double vy, double om,
                        double dt, double s0, double c0) {
  const double th1 = th + om * dt;
  if (fabs(om) >= 1e-6) {
    double s1, c1;
#if defined(__CUDA_ARCH__)
    sincos(th1, &s1, &c1);
#else
    s1 = sin(th1);
    c1 = cos(th1);
#endif
    const double s = s1 - s0;
    const double c = c1 - c0;
    x += (vx * s + vy * c) / om;
    y += (-vx * c + vy * s) / om;
  } else {
    const double half = 0.5 * om * dt * dt;
    const double ix = dt * c0 - half * s0;
    const double iy = dt * s0 + half * c0;
    x += vx * ix - vy * iy;
    y += vx * iy + vy * ix;
  }
  th = wrap_angle(th1);
}

GPM_HD void sincos_d(double a, double* s, double* c) {
#if defined(__CUDA_ARCH__)
  sincos(a, s, c);
#else
  *s = sin(a);
  *c = cos(a);
#endif
}

// dynamics.cpp:59-66 step_nominal
GPM_HD void step_nominal(const double s[5], const double u[2], const NominalDev& p, double n[5],
                         double s0, double c0) {
  double x = s[0], y = s[1], th = s[2];
  arc_advance(x, y, th, s[3], 0.0, s[4], p.dt, s0, c0);
  n[0] = x;
  n[1] = y;
  n[2] = th;
  n[3] = s[3] + (p.dt / p.tau_v) * (u[0] - s[3]);
  n[4] = s[4] + (p.dt / p.tau_omega) * (u[1] - s[4]);
}
// dynamics.cpp:100-107 step_kinematic_unicycle
GPM_HD void step_kinematic(const double s[5], const double u[2], double dt, double n[5]) {
  double x = s[0], y = s[1], th = s[2], s0, c0;
  sincos_d(th, &s0, &c0);
  arc_advance(x, y, th, u[0], 0.0, u[1], dt, s0, c0);
  n[0] = x;
  n[1] = y;
  n[2] = th;
  n[3] = u[0];
  n[4] = u[1];
}
// dynamics.cpp:109-127 step_edd5
GPM_HD void step_edd5(const double s[5], const double u[2], const Edd5Dev& p, double dt,
                      double n[5]) {
  const double span = p.y_icr_r - p.y_icr_l;
  const double wl = p.alpha_l * (u[0] - 0.5 * p.track_width * u[1]);
  const double wr = p.alpha_r * (u[0] + 0.5 * p.track_width * u[1]);
  const double om = (wr - wl) / span;
  const double v = (wr * p.y_icr_r - wl * p.y_icr_l) / span;
  const double vy = p.x_icr * om;
  double x = s[0], y = s[1], th = s[2], s0, c0;
  sincos_d(th, &s0, &c0);
  arc_advance(x, y, th, v, vy, om, dt, s0, c0);
  n[0] = x;
  n[1] = y;
  n[2] = th;
  n[3] = v;
  n[4] = om;
}
// dynamics.cpp:68-98 jacobian_nominal (row-major 5×5)
GPM_HD void jacobian_nominal(const double s[5], const NominalDev& p, double J[25]) {
  const double dt = p.dt;
  for (int i = 0; i < 25; ++i) J[i] = (i % 6 == 0) ? 1.0 : 0.0;
  const double th = s[2], v = s[3], om = s[4];
  if (fabs(om) >= 1e-6) {
    const double th1 = th + om * dt;
    double s1, c1, s0, c0;
    sincos_d(th1, &s1, &c1);
    sincos_d(th, &s0, &c0);
    const double ds = s1 - s0;
    const double dc = c1 - c0;
    const double vw = v / om;
    J[0 * 5 + 2] = vw * dc;
    J[0 * 5 + 3] = ds / om;
    J[0 * 5 + 4] = vw * dt * c1 - (v / (om * om)) * ds;
    J[1 * 5 + 2] = vw * ds;
    J[1 * 5 + 3] = -dc / om;
    J[1 * 5 + 4] = vw * dt * s1 + (v / (om * om)) * dc;
  } else {
    double s0, c0;
    sincos_d(th, &s0, &c0);
    const double half = 0.5 * om * dt * dt;
    J[0 * 5 + 2] = v * (-dt * s0 - half * c0);
    J[0 * 5 + 3] = dt * c0 - half * s0;
    J[0 * 5 + 4] = -0.5 * v * dt * dt * s0;
    J[1 * 5 + 2] = v * (dt * c0 - half * s0);
    J[1 * 5 + 3] = dt * s0 + half * c0;
    J[1 * 5 + 4] = 0.5 * v * dt * dt * c0;
  }
  J[2 * 5 + 4] = dt;
  J[3 * 5 + 3] = 1.0 - dt / p.tau_v;
  J[4 * 5 + 4] = 1.0 - dt / p.tau_omega;
}

GPM_HD bool finite5(const double s[5]) {
  return isfinite(s[0]) && isfinite(s[1]) && isfinite(s[2]) && isfinite(s[3]) && isfinite(s[4]);
}
GPM_HD double clampd(double v, double lo, double hi) { return v < lo ? lo : (hi < v ? hi : v); }

// costs.cpp:9-16 point_segment_distance
GPM_HD double point_segment(double px, double py, double ax, double ay, double bx, double by) {
  const double abx = bx - ax, aby = by - ay;
  const double len2 = abx * abx + aby * aby;
  if (len2 <= 0.0) return sqrt((px - ax) * (px - ax) + (py - ay) * (py - ay));
  double t = ((px - ax) * abx + (py - ay) * aby) / len2;
  t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
  const double ex = px - (ax + t * abx), ey = py - (ay + t * aby);
  return sqrt(ex * ex + ey * ey);
}
// costs.cpp:62-74 Track::centerline_distance (lowest segment index wins ties)
GPM_HD double centerline_distance(const TaskDev& t, double x, double y) {
  if (t.is_circle) {
    const double dx = x - t.cx, dy = y - t.cy;
    return fabs(sqrt(dx * dx + dy * dy) - t.radius);
  }
  double best = INFINITY;
  const int n = t.n_wp;
  const int nseg = t.closed ? n : n - 1;
  for (int i = 0; i < nseg; ++i) {
    const int j = (i + 1) == n ? 0 : i + 1;
    const double d = point_segment(x, y, t.wp[i][0], t.wp[i][1], t.wp[j][0], t.wp[j][1]);
    if (d < best) best = d;
  }
  return best;
}
// costs.cpp:99-102 + core.hpp:117-126 (cos/sin of prev.theta passed in)
GPM_HD double slip_ratio(const double a[5], const double b[5], double sa, double ca) {
  const double dx = b[0] - a[0], dy = b[1] - a[1];
  const double lon = ca * dx + sa * dy, lat = -sa * dx + ca * dy;
  const double den = fabs(lon) > 1e-3 ? fabs(lon) : 1e-3;
  return fabs(lat) / den;
}
// costs.cpp:104-114 collision_indicator with tightened margins
GPM_HD bool collides(const TaskDev& t, double x, double y, const double* margins_k) {
  for (int i = 0; i < t.n_obs; ++i) {
    const double dx = x - t.obs[i][0], dy = y - t.obs[i][1];
    const double s = dx * dx + dy * dy;
    // far obstacle: s > 4R^2 (R = radius + margin > 0) gives sqrt(s) - r - m >= R(1 - 1e-15) > 0,
    // the same "no collision" the exact test below returns, without the FP64 sqrt
    const double R = t.obs[i][2] + margins_k[i];
    if (R > 0.0 && s > 4.0 * R * R) continue;
    const double d = sqrt(s) - t.obs[i][2];
    if (d - margins_k[i] <= 0.0) return true;
  }
  return false;
}

// Per-step cost terms EXCLUDING the variance term (added by the variance phase):
// tracking_cost (costs.cpp:127-149) / avoidance_cost (:151-171) / combined.
struct StepCost {
  double cost;
  bool viol, coll;
};
GPM_HD StepCost step_cost(const TaskDev& t, const double prev[5], const double nx[5], double sp,
                          double cp, double r_bar_k, const double* margins_k, double v_sampled,
                          double decay) {
  StepCost out{0.0, false, false};
  if (t.kind != TASK_AVOIDANCE) {
    const double dist = centerline_distance(t, nx[0], nx[1]);
    out.viol = dist > r_bar_k;  // costs.cpp:95-97 (boundary inclusive)
    out.cost += t.tw[1] * (dist / t.half_width);
    out.cost += t.tw[2] * slip_ratio(prev, nx, sp, cp);
    out.cost += t.tw[3] * decay * (out.viol ? 1.0 : 0.0);
    const double under = t.v_desired - v_sampled;
    out.cost += t.tw[4] * (under > 0.0 ? under : 0.0);
  }
  if (t.kind != TASK_TRACKING && t.n_obs > 0) {
    out.coll = collides(t, nx[0], nx[1], margins_k);
    out.cost += t.aw[1] * (out.coll ? 1.0 : 0.0);
  }
  if (t.kind == TASK_AVOIDANCE) {
    const double gx = nx[0] - t.goal[0], gy = nx[1] - t.goal[1];
    out.cost += t.aw[2] * sqrt(gx * gx + gy * gy);
  }
  return out;
}
// variance weight of the active task (alpha0 / beta0)
GPM_HD double variance_weight(const TaskDev& t) {
  return t.kind == TASK_AVOIDANCE ? t.aw[0] : t.tw[0];
}

// ---------------------------------------------------------------------------
// Philox4x32-10 counter-based sampler (production noise; north star). Keyed by
// (seed, tick), counter = (global sample, step): independent of how samples are
// split across threads, blocks or GPUs, like the reference's per-sample
// substreams (mppi.cpp:53-62, SPEC determinism contract).
GPM_HD uint64_t splitmix64(uint64_t x) {  // rng.hpp:11-16
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
GPM_HD void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}
GPM_HD uint64_t philox_key(uint64_t seed, uint64_t tick) {
  return splitmix64(seed ^ splitmix64(tick ^ 0x6a09e667f3bcc909ULL));
}
// Standard-normal pair for (key, sample, step): Box–Muller on two 53-bit
// uniforms, FP64 (same transform as rng.hpp:45-51). Deterministic and identical
// wherever it is evaluated (rollout, update, materialisation).
GPM_HD void philox_gaussian_pair(uint64_t key, uint64_t sample, uint32_t step, double* z1,
                                 double* z2) {
  uint32_t c[4] = {(uint32_t)sample, (uint32_t)(sample >> 32), step, 0x243F6A88u};
  philox4x32_10(c, (uint32_t)key, (uint32_t)(key >> 32));
  const uint64_t a = ((uint64_t)c[1] << 32) | c[0];
  const uint64_t b = ((uint64_t)c[3] << 32) | c[2];
  const double u1 = 1.0 - (double)(a >> 11) * 0x1.0p-53;  // (0, 1]
  const double u2 = (double)(b >> 11) * 0x1.0p-53;
  const double r = sqrt(-2.0 * log(u1));
  double s, co;
#if defined(__CUDA_ARCH__)
  sincospi(2.0 * u2, &s, &co);
#else
  s = sin(2.0 * kPi * u2);
  co = cos(2.0 * kPi * u2);
#endif
  *z1 = r * co;
  *z2 = r * s;
}

// ---------------------------------------------------------------------------
// Reduction tuple: per shard, with e_s = exp(-(c_s - m)/lambda)
// over finite costs:  [m, Z=Σe, E2=Σe², H=Σe(c-m), N=#finite, C=Σc, S[T][2]=Σe·ε]
constexpr int kTupleHead = 6;
GPM_HD int tuple_doubles(int T) { return kTupleHead + 2 * T; }

// Combine n tuples in index order into out (log-sum-exp rescale to the global min).
GPM_HD void combine_tuples(const double* tuples, int n, int T, double lambda, double* out) {
  const int W = tuple_doubles(T);
  double m = INFINITY;
  for (int g = 0; g < n; ++g) {
    const double mg = tuples[(size_t)g * W + 0];
    if (mg < m) m = mg;
  }
  double Z = 0.0, E2 = 0.0, H = 0.0, N = 0.0, Csum = 0.0;
  for (int r = 0; r < 2 * T; ++r) out[kTupleHead + r] = 0.0;
  for (int g = 0; g < n; ++g) {
    const double* t = tuples + (size_t)g * W;
    N += t[4];
    Csum += t[5];
    if (!(t[4] > 0.0)) continue;  // shard without finite costs
    const double sc = exp(-(t[0] - m) / lambda);
    Z += sc * t[1];
    E2 += sc * sc * t[2];
    H += sc * (t[3] + (t[0] - m) * t[1]);
    for (int r = 0; r < 2 * T; ++r) out[kTupleHead + r] += sc * t[kTupleHead + r];
  }
  out[0] = m;
  out[1] = Z;
  out[2] = E2;
  out[3] = H;
  out[4] = N;
  out[5] = Csum;
}

}  // namespace gpm
