/*
 * gpmppi_oracle.c — FP64 CPU restatement of the reference GP-MPPI solve path.
 *
 * TEST INFRASTRUCTURE ONLY (parity checker + "port" CPU baseline). See the
 * header for the rules. Citations: /root/reference/proj/<file>:<line>.
 *
 * Threading follows the reference: fixed 128-sample chunks, chunk c handled by
 * worker c mod n_threads, threads == 0 → all host cores (mppi.cpp:15-21,
 * 401-426). Results are independent of the thread count by construction
 * (per-sample noise streams, per-index cost slots).
 */
#define _GNU_SOURCE
#include "gpmppi_oracle.h"

#include <math.h>
#include <dlfcn.h>
#include <pthread.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#include <unistd.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif
static const double kPi = 3.14159265358979323846; /* core.hpp:14 */

static __thread char g_err[512];
const char* orc_last_error(void) { return g_err; }
static int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}

/* ======================= rng.hpp:11-68 ======================= */
uint64_t orc_splitmix64(uint64_t x) { /* rng.hpp:11-16 */
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
uint64_t orc_derive_seed(uint64_t seed, uint64_t a, uint64_t b) { /* rng.hpp:19-24 */
  uint64_t h = orc_splitmix64(seed ^ 0x6a09e667f3bcc909ULL);
  h = orc_splitmix64(h ^ (a * 0x9e3779b97f4a7c15ULL));
  h = orc_splitmix64(h ^ (b * 0xbf58476d1ce4e5b9ULL));
  return h;
}
/* std::mt19937_64 (rng.hpp:26-32, 65): the C++ standard pins its parameters
 * (w=64 n=312 m=156 r=31 a=0xb5026f5aa96619e9 u=29 d=0x5555555555555555 s=17
 * b=0x71d67fffeda60000 t=37 c=0xfff7eee000000000 l=43 f=6364136223846793005). */
void orc_rng_seed(orc_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->mti = 312;
  r->has_spare = 0;
  r->spare = 0.0;
}
uint64_t orc_rng_next(orc_rng* r) {
  const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL, A = 0xB5026F5AA96619E9ULL;
  if (r->mti >= 312) {
    int i;
    for (i = 0; i < 312 - 156; ++i) {
      uint64_t x = (r->mt[i] & UM) | (r->mt[i + 1] & LM);
      r->mt[i] = r->mt[i + 156] ^ (x >> 1) ^ ((x & 1ULL) ? A : 0ULL);
    }
    for (; i < 311; ++i) {
      uint64_t x = (r->mt[i] & UM) | (r->mt[i + 1] & LM);
      r->mt[i] = r->mt[i + (156 - 312)] ^ (x >> 1) ^ ((x & 1ULL) ? A : 0ULL);
    }
    uint64_t x = (r->mt[311] & UM) | (r->mt[0] & LM);
    r->mt[311] = r->mt[155] ^ (x >> 1) ^ ((x & 1ULL) ? A : 0ULL);
    r->mti = 0;
  }
  uint64_t y = r->mt[r->mti++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= (y >> 43);
  return y;
}
double orc_rng_uniform01(orc_rng* r) { /* rng.hpp:34 */
  return (double)(orc_rng_next(r) >> 11) * 0x1.0p-53;
}
double orc_rng_uniform(orc_rng* r, double lo, double hi) { /* rng.hpp:36 */
  return lo + (hi - lo) * orc_rng_uniform01(r);
}
void orc_rng_gaussian_pair(orc_rng* r, double* z1, double* z2) { /* rng.hpp:45-51 */
  double u1 = 1.0 - orc_rng_uniform01(r);
  double u2 = orc_rng_uniform01(r);
  double rad = sqrt(-2.0 * log(u1));
  double a = 2.0 * M_PI * u2;
  *z1 = rad * cos(a);
  *z2 = rad * sin(a);
}
double orc_rng_gaussian(orc_rng* r) { /* rng.hpp:53-61 */
  if (r->has_spare) {
    r->has_spare = 0;
    return r->spare;
  }
  double z0, z1;
  orc_rng_gaussian_pair(r, &z0, &z1);
  r->spare = z1;
  r->has_spare = 1;
  return z0;
}
void orc_uniform_stream(uint64_t seed, int n, double* out) {
  orc_rng r;
  orc_rng_seed(&r, seed);
  for (int i = 0; i < n; ++i) out[i] = orc_rng_uniform01(&r);
}
void orc_gaussian_stream(uint64_t seed, int n, double* out) {
  orc_rng r;
  orc_rng_seed(&r, seed);
  for (int i = 0; i < n; ++i) out[i] = orc_rng_gaussian(&r);
}
/* mppi.cpp:53-62 fill_perturbations, one sample */
static void fill_perturbations(double* e, int T, double sv, double sw, uint64_t seed,
                               uint64_t tick, uint64_t sample) {
  orc_rng rng;
  orc_rng_seed(&rng, orc_derive_seed(seed, tick, sample));
  for (int k = 0; k < T; ++k) {
    double z1, z2;
    orc_rng_gaussian_pair(&rng, &z1, &z2);
    e[2 * k] = sv * z1;
    e[2 * k + 1] = sw * z2;
  }
}
void orc_sample_perturbations(int K, int T, double sv2, double sw2, uint64_t seed, uint64_t tick,
                              double* eps) { /* mppi.cpp:113-123 */
  const double sv = sqrt(sv2), sw = sqrt(sw2);
  for (int s = 0; s < K; ++s)
    fill_perturbations(eps + (size_t)s * T * 2, T, sv, sw, seed, tick, (uint64_t)s);
}

/* ======================= core.hpp / dynamics.cpp ======================= */
static int finite5(const double s[5]) {
  return isfinite(s[0]) && isfinite(s[1]) && isfinite(s[2]) && isfinite(s[3]) && isfinite(s[4]);
}
double orc_wrap_angle(double a) { /* core.hpp:18-27 */
  double r = remainder(a, 2.0 * kPi);
  if (r <= -kPi) r += 2.0 * kPi;
  return r;
}
void orc_arc_advance(double* x, double* y, double* th, double vx, double vy, double om,
                     double dt) { /* dynamics.cpp:39-57 */
  if (fabs(om) >= 1e-6) {
    const double s = sin(*th + om * dt) - sin(*th);
    const double c = cos(*th + om * dt) - cos(*th);
    *x += (vx * s + vy * c) / om;
    *y += (-vx * c + vy * s) / om;
  } else {
    const double c0 = cos(*th), s0 = sin(*th);
    const double half = 0.5 * om * dt * dt;
    const double ix = dt * c0 - half * s0;
    const double iy = dt * s0 + half * c0;
    *x += vx * ix - vy * iy;
    *y += vx * iy + vy * ix;
  }
  *th = orc_wrap_angle(*th + om * dt);
}
void orc_step_nominal(const double s[5], const double u[2], const orc_nominal* p,
                      double n[5]) { /* dynamics.cpp:59-66 */
  double x = s[0], y = s[1], th = s[2];
  orc_arc_advance(&x, &y, &th, s[3], 0.0, s[4], p->dt);
  n[0] = x;
  n[1] = y;
  n[2] = th;
  n[3] = s[3] + (p->dt / p->tau_v) * (u[0] - s[3]);
  n[4] = s[4] + (p->dt / p->tau_omega) * (u[1] - s[4]);
}
void orc_jacobian_nominal(const double s[5], const double u[2], const orc_nominal* p,
                          double J[25]) { /* dynamics.cpp:68-98 */
  (void)u;
  const double dt = p->dt;
  for (int i = 0; i < 25; ++i) J[i] = (i % 6 == 0) ? 1.0 : 0.0;
  const double th = s[2], v = s[3], om = s[4];
  if (fabs(om) >= 1e-6) {
    const double th1 = th + om * dt;
    const double ds = sin(th1) - sin(th);
    const double dc = cos(th1) - cos(th);
    const double vw = v / om;
    J[0 * 5 + 2] = vw * dc;
    J[0 * 5 + 3] = ds / om;
    J[0 * 5 + 4] = vw * dt * cos(th1) - (v / (om * om)) * ds;
    J[1 * 5 + 2] = vw * ds;
    J[1 * 5 + 3] = -dc / om;
    J[1 * 5 + 4] = vw * dt * sin(th1) + (v / (om * om)) * dc;
  } else {
    const double c0 = cos(th), s0 = sin(th);
    const double half = 0.5 * om * dt * dt;
    J[0 * 5 + 2] = v * (-dt * s0 - half * c0);
    J[0 * 5 + 3] = dt * c0 - half * s0;
    J[0 * 5 + 4] = -0.5 * v * dt * dt * s0;
    J[1 * 5 + 2] = v * (dt * c0 - half * s0);
    J[1 * 5 + 3] = dt * s0 + half * c0;
    J[1 * 5 + 4] = 0.5 * v * dt * dt * c0;
  }
  J[2 * 5 + 4] = dt;
  J[3 * 5 + 3] = 1.0 - dt / p->tau_v;
  J[4 * 5 + 4] = 1.0 - dt / p->tau_omega;
}
void orc_step_kinematic(const double s[5], const double u[2], double dt,
                        double n[5]) { /* dynamics.cpp:100-107 */
  double x = s[0], y = s[1], th = s[2];
  orc_arc_advance(&x, &y, &th, u[0], 0.0, u[1], dt);
  n[0] = x;
  n[1] = y;
  n[2] = th;
  n[3] = u[0];
  n[4] = u[1];
}
void orc_step_edd5(const double s[5], const double u[2], const orc_edd5* p, double track_width,
                   double dt, double n[5]) { /* dynamics.cpp:109-127 */
  const double span = p->y_icr_r - p->y_icr_l;
  const double wl = p->alpha_l * (u[0] - 0.5 * track_width * u[1]);
  const double wr = p->alpha_r * (u[0] + 0.5 * track_width * u[1]);
  const double om = (wr - wl) / span;
  const double v = (wr * p->y_icr_r - wl * p->y_icr_l) / span;
  const double vy = p->x_icr * om;
  double x = s[0], y = s[1], th = s[2];
  orc_arc_advance(&x, &y, &th, v, vy, om, dt);
  n[0] = x;
  n[1] = y;
  n[2] = th;
  n[3] = v;
  n[4] = om;
}

/* ======================= gp.cpp ======================= */
typedef struct {
  double kernel[6]; /* signal_var, ls[4], noise_var */
  int n_out;
  int outputs[64];
  double* inputs_aug;  /* n×6: [x/l | 1 | -0.5|x/l|^2 + ln sv]  gp.cpp:103-110 */
  double* chol;        /* n×n lower */
  double* inv_lower_t; /* n×n upper (row-major) */
  double* alphas;      /* n×n_out */
  double jitter;
} orc_group;
struct orc_gp {
  int n, m, n_groups;
  orc_group groups[64];
  double* lml;
};

double orc_kernel_eval(const double a[4], const double b[4], const double k6[6]) {
  /* gp.cpp:53-59 */
  double s = 0.0;
  for (int d = 0; d < 4; ++d) {
    const double t = (a[d] - b[d]) / k6[1 + d];
    s += t * t;
  }
  return k6[0] * exp(-0.5 * s);
}

/* Eigen LLT semantics: fails iff a pivot is <= 0 (Eigen/src/Cholesky/LLT.h). */
static int cholesky_lower(double* A, int n) {
  for (int j = 0; j < n; ++j) {
    double x = A[(size_t)j * n + j];
    for (int k = 0; k < j; ++k) x -= A[(size_t)j * n + k] * A[(size_t)j * n + k];
    if (!(x > 0.0)) return -1;
    const double d = sqrt(x);
    A[(size_t)j * n + j] = d;
    for (int i = j + 1; i < n; ++i) {
      double v = A[(size_t)i * n + j];
      const double* ri = A + (size_t)i * n;
      const double* rj = A + (size_t)j * n;
      for (int k = 0; k < j; ++k) v -= ri[k] * rj[k];
      A[(size_t)i * n + j] = v / d;
    }
  }
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j) A[(size_t)i * n + j] = 0.0;
  return 0;
}

int orc_gp_fit(const double* X, const double* Y, int n, int m, const double* kernels,
               orc_gp** out) { /* gp.cpp:61-150 */
  *out = NULL;
  if (n < 1) return fail(ORC_INVALID_ARGUMENT, "GpModel::fit: inputs must be n x 4 with n >= 1");
  if (m < 1) return fail(ORC_INVALID_ARGUMENT, "GpModel::fit: outputs must be n x m with m >= 1");
  for (size_t i = 0; i < (size_t)n * 4; ++i)
    if (!isfinite(X[i])) return fail(ORC_INVALID_ARGUMENT, "GpModel::fit: non-finite training data");
  for (size_t i = 0; i < (size_t)n * m; ++i)
    if (!isfinite(Y[i])) return fail(ORC_INVALID_ARGUMENT, "GpModel::fit: non-finite training data");
  orc_gp* g = (orc_gp*)calloc(1, sizeof(orc_gp));
  g->n = n;
  g->m = m;
  g->lml = (double*)calloc((size_t)m, sizeof(double));
  for (int j = 0; j < m; ++j) { /* gp.cpp:85-100 grouping */
    const double* kp = kernels + 6 * j;
    int ok = kp[0] > 0.0 && kp[5] > 0.0;
    for (int d = 0; d < 4; ++d) ok = ok && kp[1 + d] > 0.0;
    if (!ok) {
      orc_gp_free(g);
      return fail(ORC_INVALID_ARGUMENT, "KernelParams: all parameters must be strictly positive");
    }
    int grp = -1;
    for (int k = 0; k < g->n_groups; ++k)
      if (memcmp(g->groups[k].kernel, kp, 6 * sizeof(double)) == 0) {
        grp = k;
        break;
      }
    if (grp < 0) {
      grp = g->n_groups++;
      memcpy(g->groups[grp].kernel, kp, 6 * sizeof(double));
    }
    g->groups[grp].outputs[g->groups[grp].n_out++] = j;
  }
  const double log2pi = log(2.0 * kPi);
  for (int gi = 0; gi < g->n_groups; ++gi) {
    orc_group* G = &g->groups[gi];
    const double sv = G->kernel[0], nv = G->kernel[5];
    G->inputs_aug = (double*)malloc(sizeof(double) * (size_t)n * 6);
    double* norms = (double*)malloc(sizeof(double) * (size_t)n);
    for (int i = 0; i < n; ++i) {
      double sq = 0.0;
      for (int d = 0; d < 4; ++d) {
        const double v = X[(size_t)i * 4 + d] / G->kernel[1 + d];
        G->inputs_aug[(size_t)i * 6 + d] = v;
        sq += v * v;
      }
      norms[i] = -0.5 * sq;
      G->inputs_aug[(size_t)i * 6 + 4] = 1.0;
      G->inputs_aug[(size_t)i * 6 + 5] = norms[i] + log(sv);
    }
    /* gp.cpp:112-114 K_ij = exp(a_i.b_j + an_i + bn_j), symmetrised */
    double* K = (double*)malloc(sizeof(double) * (size_t)n * n);
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        double dot = 0.0;
        for (int d = 0; d < 4; ++d)
          dot += G->inputs_aug[(size_t)i * 6 + d] * G->inputs_aug[(size_t)j * 6 + d];
        K[(size_t)i * n + j] = exp(dot + norms[i] + G->inputs_aug[(size_t)j * 6 + 5]);
      }
    for (int i = 0; i < n; ++i)
      for (int j = i + 1; j < n; ++j) {
        const double s = 0.5 * (K[(size_t)i * n + j] + K[(size_t)j * n + i]);
        K[(size_t)i * n + j] = s;
        K[(size_t)j * n + i] = s;
      }
    /* gp.cpp:116-133 jitter ladder */
    double* L = (double*)malloc(sizeof(double) * (size_t)n * n);
    int ok = 0;
    double jitter = 0.0;
    for (int attempt = 0; attempt <= 5 && !ok; ++attempt) {
      jitter = attempt == 0 ? 0.0 : pow(10.0, -11 + attempt);
      memcpy(L, K, sizeof(double) * (size_t)n * n);
      for (int i = 0; i < n; ++i) L[(size_t)i * n + i] += nv + jitter;
      ok = cholesky_lower(L, n) == 0;
    }
    free(K);
    free(norms);
    if (!ok) {
      free(L);
      orc_gp_free(g);
      return fail(ORC_RUNTIME_ERROR,
                  "GpModel::fit: Cholesky failed for kernel group after jitter up to 1e-6 "
                  "(signal_var=%g, noise_var=%g)",
                  sv, nv);
    }
    G->jitter = jitter;
    G->chol = L;
    /* gp.cpp:135-138 L^{-T} via forward substitution on the identity */
    double* Xinv = (double*)calloc((size_t)n * n, sizeof(double)); /* L^{-1}, lower */
    for (int c = 0; c < n; ++c) {
      for (int i = c; i < n; ++i) {
        double v = (i == c) ? 1.0 : 0.0;
        for (int k = c; k < i; ++k) v -= L[(size_t)i * n + k] * Xinv[(size_t)k * n + c];
        Xinv[(size_t)i * n + c] = v / L[(size_t)i * n + i];
      }
    }
    G->inv_lower_t = (double*)calloc((size_t)n * n, sizeof(double));
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) G->inv_lower_t[(size_t)i * n + j] = Xinv[(size_t)j * n + i];
    free(Xinv);
    /* gp.cpp:140-147 alphas and LML */
    G->alphas = (double*)malloc(sizeof(double) * (size_t)n * G->n_out);
    double logdet = 0.0;
    for (int i = 0; i < n; ++i) logdet += log(L[(size_t)i * n + i]);
    double* z = (double*)malloc(sizeof(double) * (size_t)n);
    for (int c = 0; c < G->n_out; ++c) {
      const int j = G->outputs[c];
      for (int i = 0; i < n; ++i) {
        double v = Y[(size_t)i * m + j];
        for (int k = 0; k < i; ++k) v -= L[(size_t)i * n + k] * z[k];
        z[i] = v / L[(size_t)i * n + i];
      }
      for (int i = n - 1; i >= 0; --i) {
        double v = z[i];
        for (int k = i + 1; k < n; ++k) v -= L[(size_t)k * n + i] * G->alphas[(size_t)k * G->n_out + c];
        G->alphas[(size_t)i * G->n_out + c] = v / L[(size_t)i * n + i];
      }
      double dot = 0.0;
      for (int i = 0; i < n; ++i) dot += Y[(size_t)i * m + j] * G->alphas[(size_t)i * G->n_out + c];
      g->lml[j] = -0.5 * dot - logdet - 0.5 * (double)n * log2pi;
    }
    free(z);
  }
  *out = g;
  return ORC_OK;
}
void orc_gp_free(orc_gp* g) {
  if (!g) return;
  for (int i = 0; i < g->n_groups; ++i) {
    free(g->groups[i].inputs_aug);
    free(g->groups[i].chol);
    free(g->groups[i].inv_lower_t);
    free(g->groups[i].alphas);
  }
  free(g->lml);
  free(g);
}
int orc_gp_n_points(const orc_gp* g) { return g->n; }
int orc_gp_n_outputs(const orc_gp* g) { return g->m; }
int orc_gp_n_groups(const orc_gp* g) { return g->n_groups; }
double orc_gp_group_jitter(const orc_gp* g, int grp) { return g->groups[grp].jitter; }
double orc_gp_lml(const orc_gp* g, int o) { return g->lml[o]; }
void orc_gp_group_export(const orc_gp* g, int grp, double* ilt, double* chol, double* alphas,
                         double* aug, int* outputs, int* n_out, double* kernel6) {
  const orc_group* G = &g->groups[grp];
  const size_t n = (size_t)g->n;
  if (ilt) memcpy(ilt, G->inv_lower_t, sizeof(double) * n * n);
  if (chol) memcpy(chol, G->chol, sizeof(double) * n * n);
  if (alphas) memcpy(alphas, G->alphas, sizeof(double) * n * G->n_out);
  if (aug) memcpy(aug, G->inputs_aug, sizeof(double) * n * 6);
  if (outputs) memcpy(outputs, G->outputs, sizeof(int) * G->n_out);
  if (n_out) *n_out = G->n_out;
  if (kernel6) memcpy(kernel6, G->kernel, sizeof(double) * 6);
}

/* Optional BLAS for the timed CPU baseline (bench.py's reference arm only; the parity
 * checker keeps the scalar loops below). The reference evaluates the kernel row, the
 * mean and the variance with Eigen GEMM / GEMM / TRMM (gp.cpp:178, 182, 185); an
 * optimised BLAS (OpenBLAS, loaded with dlopen) stands in for Eigen's kernels, which
 * cannot be built here (no Eigen in the image). Single-threaded BLAS inside each of the
 * reference's per-chunk worker threads, as Eigen runs there. */
typedef void (*orc_dgemm_fn)(int, int, int, int, int, int, double, const double*, int,
                             const double*, int, double, double*, int);
typedef void (*orc_dtrmm_fn)(int, int, int, int, int, int, int, double, const double*, int,
                             double*, int);
static orc_dgemm_fn g_dgemm = NULL;
static orc_dtrmm_fn g_dtrmm = NULL;
enum { CB_ROW = 101, CB_NOTRANS = 111, CB_TRANS = 112, CB_UPPER = 121, CB_NONUNIT = 131,
       CB_RIGHT = 142 };

int orc_use_blas(const char* so_path, const char* prefix) {
  if (!so_path) {
    g_dgemm = NULL;
    g_dtrmm = NULL;
    return 0;
  }
  void* h = dlopen(so_path, RTLD_NOW | RTLD_LOCAL);
  if (!h) return -1;
  char name[128];
  snprintf(name, sizeof name, "%scblas_dgemm", prefix ? prefix : "");
  orc_dgemm_fn gm = (orc_dgemm_fn)dlsym(h, name);
  snprintf(name, sizeof name, "%scblas_dtrmm", prefix ? prefix : "");
  orc_dtrmm_fn tm = (orc_dtrmm_fn)dlsym(h, name);
  snprintf(name, sizeof name, "%sopenblas_set_num_threads", prefix ? prefix : "");
  void (*nt)(int) = (void (*)(int))dlsym(h, name);
  if (!gm || !tm) return -2;
  if (nt) nt(1);
  g_dgemm = gm;
  g_dtrmm = tm;
  return 0;
}

/* gp.cpp:152-198 with the BLAS stand-in for Eigen: K* = exp(Q_aug · aug^T) (GEMM),
 * mean = K* · alphas (GEMM), a = K* · L^{-T} (TRMM), var = max(sv - |a|^2, 0). */
static void predict_block_blas(const orc_gp* g, const double* q, int S, double* mean,
                               double* var, double* ws) {
  const int n = g->n, m = g->m;
  double* kstar = ws;
  double* a = ws + (size_t)S * n;
  double qa[6 * 128];
  double mo[8 * 128];
  for (int gi = 0; gi < g->n_groups; ++gi) {
    const orc_group* G = &g->groups[gi];
    for (int s0 = 0; s0 < S; s0 += 128) {
      const int cs = (S - s0) < 128 ? (S - s0) : 128;
      for (int s = 0; s < cs; ++s) {
        double sq = 0.0;
        for (int d = 0; d < 4; ++d) {
          qa[s * 6 + d] = q[(size_t)(s0 + s) * 4 + d] / G->kernel[1 + d];
          sq += qa[s * 6 + d] * qa[s * 6 + d];
        }
        qa[s * 6 + 4] = -0.5 * sq;
        qa[s * 6 + 5] = 1.0;
      }
      double* kr = kstar + (size_t)s0 * n;
      g_dgemm(CB_ROW, CB_NOTRANS, CB_TRANS, cs, n, 6, 1.0, qa, 6, G->inputs_aug, 6, 0.0, kr, n);
      for (size_t i = 0; i < (size_t)cs * n; ++i) kr[i] = exp(kr[i]);
      for (int c0 = 0; c0 < G->n_out; c0 += 8) {
        const int nc = (G->n_out - c0) < 8 ? (G->n_out - c0) : 8;
        g_dgemm(CB_ROW, CB_NOTRANS, CB_NOTRANS, cs, nc, n, 1.0, kr, n, G->alphas + c0, G->n_out, 0.0,
                mo, nc);
        for (int s = 0; s < cs; ++s)
          for (int c = 0; c < nc; ++c) mean[(size_t)(s0 + s) * m + G->outputs[c0 + c]] = mo[s * nc + c];
      }
    }
    memcpy(a, kstar, sizeof(double) * (size_t)S * n);
    g_dtrmm(CB_ROW, CB_RIGHT, CB_UPPER, CB_NOTRANS, CB_NONUNIT, S, n, 1.0, G->inv_lower_t, n, a, n);
    for (int s = 0; s < S; ++s) {
      double v = G->kernel[0];
      const double* ar = a + (size_t)s * n;
      for (int j = 0; j < n; ++j) v -= ar[j] * ar[j];
      v = v > 0.0 ? v : 0.0;
      for (int c = 0; c < G->n_out; ++c) var[(size_t)s * m + G->outputs[c]] = v;
    }
  }
}

/* gp.cpp:152-198 for S queries (row-major S×4) into mean/var (S×m).
 * ws must hold S*n*2 doubles. The TRMM is blocked 8 rows of L^{-T} at a time so
 * the inner loop streams contiguous rows (vectorisable at -O3). */
static void predict_block(const orc_gp* g, const double* q, int S, double* mean, double* var,
                          double* ws) {
  const int n = g->n, m = g->m;
  double* kstar = ws;
  double* a = ws + (size_t)S * n;
  if (g_dgemm && g_dtrmm) {
    predict_block_blas(g, q, S, mean, var, ws);
    return;
  }
  for (int gi = 0; gi < g->n_groups; ++gi) {
    const orc_group* G = &g->groups[gi];
    const double* aug = G->inputs_aug;
    for (int s = 0; s < S; ++s) {
      double qa[6];
      double sq = 0.0;
      for (int d = 0; d < 4; ++d) {
        qa[d] = q[(size_t)s * 4 + d] / G->kernel[1 + d];
        sq += qa[d] * qa[d];
      }
      qa[4] = -0.5 * sq;
      qa[5] = 1.0;
      double* kr = kstar + (size_t)s * n;
      for (int j = 0; j < n; ++j) {
        const double* z = aug + (size_t)j * 6;
        const double dot = qa[0] * z[0] + qa[1] * z[1] + qa[2] * z[2] + qa[3] * z[3] +
                           qa[4] * z[4] + qa[5] * z[5];
        kr[j] = exp(dot);
      }
      for (int c = 0; c < G->n_out; ++c) {
        double acc = 0.0;
        for (int j = 0; j < n; ++j) acc += kr[j] * G->alphas[(size_t)j * G->n_out + c];
        mean[(size_t)s * m + G->outputs[c]] = acc;
      }
    }
    memset(a, 0, sizeof(double) * (size_t)S * n);
    const double* Lt = G->inv_lower_t;
    for (int i0 = 0; i0 < n; i0 += 8) {
      const int ib = (n - i0) < 8 ? (n - i0) : 8;
      for (int s = 0; s < S; ++s) {
        const double* kr = kstar + (size_t)s * n + i0;
        double* ar = a + (size_t)s * n;
        for (int jj = 0; jj < ib; ++jj) {
          const int j = i0 + jj;
          double acc = ar[j];
          for (int ii = 0; ii <= jj; ++ii) acc += kr[ii] * Lt[(size_t)(i0 + ii) * n + j];
          ar[j] = acc;
        }
        if (ib == 8) {
          const double k0 = kr[0], k1 = kr[1], k2 = kr[2], k3 = kr[3], k4 = kr[4], k5 = kr[5],
                       k6 = kr[6], k7 = kr[7];
          const double *l0 = Lt + (size_t)i0 * n, *l1 = l0 + n, *l2 = l1 + n, *l3 = l2 + n,
                       *l4 = l3 + n, *l5 = l4 + n, *l6 = l5 + n, *l7 = l6 + n;
          for (int j = i0 + 8; j < n; ++j)
            ar[j] += k0 * l0[j] + k1 * l1[j] + k2 * l2[j] + k3 * l3[j] + k4 * l4[j] +
                     k5 * l5[j] + k6 * l6[j] + k7 * l7[j];
        }
      }
    }
    for (int s = 0; s < S; ++s) {
      double v = G->kernel[0];
      const double* ar = a + (size_t)s * n;
      for (int j = 0; j < n; ++j) v -= ar[j] * ar[j]; /* gp.cpp:188-190 column order */
      v = v > 0.0 ? v : 0.0;                           /* gp.cpp:191 */
      for (int c = 0; c < G->n_out; ++c) var[(size_t)s * m + G->outputs[c]] = v;
    }
  }
}
int orc_gp_predict_batch(const orc_gp* g, const double* q, int S, double* mean, double* var) {
  if (S == 0) return ORC_OK;
  for (size_t i = 0; i < (size_t)S * 4; ++i)
    if (!isfinite(q[i])) return fail(ORC_INVALID_ARGUMENT, "GpModel::predict: non-finite query");
  double* ws = (double*)malloc(sizeof(double) * (size_t)2 * g->n * (S < 128 ? S : 128));
  for (int s0 = 0; s0 < S; s0 += 128) {
    const int cs = (S - s0) < 128 ? (S - s0) : 128;
    predict_block(g, q + (size_t)s0 * 4, cs, mean + (size_t)s0 * g->m, var + (size_t)s0 * g->m,
                  ws);
  }
  free(ws);
  return ORC_OK;
}

static int on_simplex(const double* w, int R, double tol) { /* core.hpp:107-111 */
  if (R == 0) return 0;
  double sum = 0.0;
  for (int i = 0; i < R; ++i) sum += w[i];
  if (fabs(sum - 1.0) > tol) return 0;
  for (int i = 0; i < R; ++i)
    if (!(w[i] >= -tol) || !(w[i] <= 1.0 + tol)) return 0;
  return 1;
}
/* mppi.cpp:34-49 / gp.cpp:368-389 ascending-i accumulation */
static void combine(const double* w, int R, const double* mean_row, const double* var_row,
                    double cm[2], double cv[2]) {
  double m0 = 0.0, m1 = 0.0, vv = 0.0, vw = 0.0;
  for (int i = 0; i < R; ++i) {
    const double wi = w[i];
    m0 += wi * mean_row[2 * i];
    m1 += wi * mean_row[2 * i + 1];
    vv += wi * wi * var_row[2 * i];
    vw += wi * wi * var_row[2 * i + 1];
  }
  cm[0] = m0;
  cm[1] = m1;
  cv[0] = vv;
  cv[1] = vw;
}
int orc_ensemble_combine(const double* means, const double* vars, const double* w, int R,
                         double mean[2], double cov[2]) {
  if (R < 1) return fail(ORC_INVALID_ARGUMENT, "ensemble_combine: size mismatch");
  if (!on_simplex(w, R, 1e-6))
    return fail(ORC_INVALID_ARGUMENT, "ensemble_combine: weights off the simplex beyond 1e-6");
  combine(w, R, means, vars, mean, cov);
  return ORC_OK;
}

/* mppi.cpp:80-111 rollout(): mean-only rollout of one control sequence. GP ensemble:
 * predict at (v, w, u) -> combine_terrains -> step_nominal + mean correction;
 * baselines: baseline_step (mppi.cpp:23-29); NOMINAL (repo extension): step_nominal.
 * states (T+1)x5, corr Tx4 = (mean_v, mean_w, var_v, var_w). */
int orc_rollout(int kind, const orc_gp* gp, int R, const double* w, const orc_nominal* nom,
                const orc_edd5* edd, double track_width, const double x0[5], const double* seq,
                int T, double* states, double* corr) {
  if (kind == ORC_MODEL_GP) {
    if (!gp || R < 1 || gp->m != 2 * R) return fail(ORC_INVALID_ARGUMENT, "rollout: bad GP ensemble");
    if (!on_simplex(w, R, 1e-6))
      return fail(ORC_INVALID_ARGUMENT, "rollout: terrain weights must lie on the simplex");
  }
  for (int i = 0; i < 5; ++i) states[i] = x0[i];
  double* mean = kind == ORC_MODEL_GP ? (double*)malloc(sizeof(double) * gp->m) : NULL;
  double* var = kind == ORC_MODEL_GP ? (double*)malloc(sizeof(double) * gp->m) : NULL;
  double* ws = kind == ORC_MODEL_GP ? (double*)malloc(sizeof(double) * 2 * (size_t)gp->n) : NULL;
  for (int k = 0; k < T; ++k) {
    const double* s = states + 5 * k;
    double* nx = states + 5 * (k + 1);
    const double* u = seq + 2 * k;
    double cm[2] = {0.0, 0.0}, cv[2] = {0.0, 0.0};
    if (kind == ORC_MODEL_GP) {
      const double q[4] = {s[3], s[4], u[0], u[1]};
      predict_block(gp, q, 1, mean, var, ws);
      combine(w, R, mean, var, cm, cv);
      orc_step_nominal(s, u, nom, nx);
      nx[3] += cm[0];
      nx[4] += cm[1];
    } else if (kind == ORC_MODEL_EDD5) {
      orc_step_edd5(s, u, edd, track_width, nom->dt, nx);
    } else if (kind == ORC_MODEL_UNICYCLE) {
      orc_step_kinematic(s, u, nom->dt, nx);
    } else {
      orc_step_nominal(s, u, nom, nx);
    }
    corr[4 * k] = cm[0];
    corr[4 * k + 1] = cm[1];
    corr[4 * k + 2] = cv[0];
    corr[4 * k + 3] = cv[1];
  }
  free(mean);
  free(var);
  free(ws);
  return ORC_OK;
}

/* ======================= uncertainty.cpp ======================= */
double orc_chi2_quantile_2dof(double p) { return -2.0 * log1p(-p); } /* :8-13 */
double orc_normal_cdf(double x) { return 0.5 * erfc(-x * M_SQRT1_2); } /* :15 */
static double nq_approx(double p) { /* :19-46 Acklam */
  static const double a[] = {-3.969683028665376e+01, 2.209460984245205e+02,
                             -2.759285104469687e+02, 1.383577518672690e+02,
                             -3.066479806614716e+01, 2.506628277459239e+00};
  static const double b[] = {-5.447609879822406e+01, 1.615858368580409e+02,
                             -1.556989798598866e+02, 6.680131188771972e+01,
                             -1.328068155288572e+01};
  static const double c[] = {-7.784894002430293e-03, -3.223964580411365e-01,
                             -2.400758277161838e+00, -2.549732539343734e+00,
                             4.374664141464968e+00,  2.938163982698783e+00};
  static const double d[] = {7.784695709041462e-03, 3.224671290700398e-01,
                             2.445134137142996e+00, 3.754408661907416e+00};
  const double plow = 0.02425;
  if (p < plow) {
    const double q = sqrt(-2.0 * log(p));
    return (((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
           ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1.0);
  }
  if (p > 1.0 - plow) {
    const double q = sqrt(-2.0 * log(1.0 - p));
    return -(((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
           ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1.0);
  }
  const double q = p - 0.5;
  const double r = q * q;
  return (((((a[0] * r + a[1]) * r + a[2]) * r + a[3]) * r + a[4]) * r + a[5]) * q /
         (((((b[0] * r + b[1]) * r + b[2]) * r + b[3]) * r + b[4]) * r + 1.0);
}
double orc_normal_quantile(double p) { /* :49-60 */
  double x = nq_approx(p);
  const double pdf = exp(-0.5 * x * x) / sqrt(2.0 * kPi);
  if (pdf > 1e-300) x -= (orc_normal_cdf(x) - p) / pdf;
  return x;
}
double orc_lambda_max_2x2(const double m[4]) { /* :62-66 */
  const double half_tr = 0.5 * (m[0] + m[3]);
  const double det_disc = 0.25 * (m[0] - m[3]) * (m[0] - m[3]) + m[1] * m[2];
  return half_tr + sqrt(det_disc > 0.0 ? det_disc : 0.0);
}
void orc_propagate_belief(const double mu[5], const double cov[25], const double u[2],
                          const double cm[2], const double cv[2], const orc_nominal* p,
                          double omu[5], double ocov[25]) { /* :75-88 */
  double nm[5];
  orc_step_nominal(mu, u, p, nm);
  nm[3] += cm[0];
  nm[4] += cm[1];
  double J[25], JS[25], C[25];
  orc_jacobian_nominal(mu, u, p, J);
  for (int i = 0; i < 5; ++i)
    for (int j = 0; j < 5; ++j) {
      double s = 0.0;
      for (int k = 0; k < 5; ++k) s += J[i * 5 + k] * cov[k * 5 + j];
      JS[i * 5 + j] = s;
    }
  for (int i = 0; i < 5; ++i)
    for (int j = 0; j < 5; ++j) {
      double s = 0.0;
      for (int k = 0; k < 5; ++k) s += JS[i * 5 + k] * J[j * 5 + k];
      C[i * 5 + j] = s;
    }
  C[3 * 5 + 3] += cv[0];
  C[4 * 5 + 4] += cv[1];
  for (int i = 0; i < 5; ++i)
    for (int j = 0; j < 5; ++j) ocov[i * 5 + j] = 0.5 * (C[i * 5 + j] + C[j * 5 + i]);
  memcpy(omu, nm, sizeof nm);
}
double orc_tighten_lane_radius(double r, const double cxy[4], double chi2_2) { /* :90-96 */
  double l = orc_lambda_max_2x2(cxy);
  l = l > 0.0 ? l : 0.0;
  return r - sqrt(chi2_2 * l);
}
double orc_tighten_obstacle_distance(const double xy[2], const double c[2], double radius,
                                     const double cxy[4], double z, double* d_out,
                                     double nrm[2], int* degenerate) { /* :98-116 */
  const double dx = xy[0] - c[0], dy = xy[1] - c[1];
  const double dist = sqrt(dx * dx + dy * dy);
  double d, n0, n1;
  int deg = 0;
  if (dist < 1e-12) {
    deg = 1;
    n0 = 1.0;
    n1 = 0.0;
    d = -radius;
  } else {
    n0 = dx / dist;
    n1 = dy / dist;
    d = dist - radius;
  }
  /* n.dot(cov * n) */
  const double cn0 = cxy[0] * n0 + cxy[1] * n1, cn1 = cxy[2] * n0 + cxy[3] * n1;
  double dir_var = n0 * cn0 + n1 * cn1;
  dir_var = dir_var > 0.0 ? dir_var : 0.0;
  if (d_out) *d_out = d;
  if (nrm) {
    nrm[0] = n0;
    nrm[1] = n1;
  }
  if (degenerate) *degenerate = deg;
  return d - z * sqrt(dir_var);
}

/* ======================= costs.cpp ======================= */
static double pt_seg(double px, double py, double ax, double ay, double bx,
                     double by) { /* :9-16 */
  const double abx = bx - ax, aby = by - ay;
  const double len2 = abx * abx + aby * aby;
  if (len2 <= 0.0) return sqrt((px - ax) * (px - ax) + (py - ay) * (py - ay));
  double t = ((px - ax) * abx + (py - ay) * aby) / len2;
  t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
  const double ex = px - (ax + t * abx), ey = py - (ay + t * aby);
  return sqrt(ex * ex + ey * ey);
}
double orc_centerline_distance(const orc_track* t, double x, double y) { /* :62-74 */
  if (t->is_circle) {
    const double dx = x - t->cx, dy = y - t->cy;
    return fabs(sqrt(dx * dx + dy * dy) - t->radius);
  }
  double best = INFINITY;
  const int n = t->n_waypoints;
  const int nseg = t->closed ? n : n - 1;
  for (int i = 0; i < nseg; ++i) {
    const int j = (i + 1) % n;
    const double d = pt_seg(x, y, t->waypoints[2 * i], t->waypoints[2 * i + 1],
                            t->waypoints[2 * j], t->waypoints[2 * j + 1]);
    if (d < best) best = d;
  }
  return best;
}
double orc_slip_ratio(const double a[5], const double b[5]) { /* :99-102 + core.hpp:117-126 */
  const double dx = b[0] - a[0], dy = b[1] - a[1];
  const double c = cos(a[2]), s = sin(a[2]);
  const double lon = c * dx + s * dy, lat = -s * dx + c * dy;
  const double den = fabs(lon) > 1e-3 ? fabs(lon) : 1e-3;
  return fabs(lat) / den;
}
double orc_collision_indicator(double x, double y, const double* obs, int O,
                               const double* margins) { /* :104-114 */
  for (int i = 0; i < O; ++i) {
    const double dx = x - obs[3 * i], dy = y - obs[3 * i + 1];
    const double d = sqrt(dx * dx + dy * dy) - obs[3 * i + 2];
    if (d - margins[i] <= 0.0) return 1.0;
  }
  return 0.0;
}
double orc_tracking_cost(const double* st, const double* tr, int N, const orc_track* track,
                         const double* r_bar, double v_des, const double* v_s,
                         const orc_tracking_weights* w) { /* :127-149 */
  double cost = 0.0, decay = 1.0;
  for (int k = 0; k < N; ++k) {
    const double* nx = st + 5 * (k + 1);
    const double dist = orc_centerline_distance(track, nx[0], nx[1]);
    cost += w->variance * tr[k];
    cost += w->deviation * (dist / track->half_width);
    cost += w->slip * orc_slip_ratio(st + 5 * k, nx);
    cost += w->safety * decay * (dist > r_bar[k] ? 1.0 : 0.0);
    const double sp = v_des - v_s[k];
    cost += w->speed * (sp > 0.0 ? sp : 0.0);
    decay *= 0.9;
  }
  return cost;
}
double orc_avoidance_cost(const double* st, const double* tr, int N, const double* obs, int O,
                          const double* margins, const double goal[3],
                          const orc_avoidance_weights* w, double high_cost) { /* :151-171 */
  double cost = 0.0;
  for (int k = 0; k < N; ++k) {
    const double* nx = st + 5 * (k + 1);
    cost += w->variance * tr[k];
    cost += w->obstacle * orc_collision_indicator(nx[0], nx[1], obs, O, margins + (size_t)k * O);
    const double gx = nx[0] - goal[0], gy = nx[1] - goal[1];
    cost += w->stage * sqrt(gx * gx + gy * gy);
  }
  const double* last = st + 5 * N;
  const double gx = last[0] - goal[0], gy = last[1] - goal[1];
  cost += w->terminal * (sqrt(gx * gx + gy * gy) <= goal[2] ? 0.0 : high_cost);
  return cost;
}

/* ======================= mppi.cpp ======================= */
void orc_trajectory_weights(const double* c, int K, double lambda, double* w) { /* :125-145 */
  double lo = INFINITY;
  for (int i = 0; i < K; ++i) {
    w[i] = 0.0;
    if (isfinite(c[i])) lo = c[i] < lo ? c[i] : lo;
  }
  if (!isfinite(lo)) return;
  double sum = 0.0;
  for (int i = 0; i < K; ++i)
    if (isfinite(c[i])) {
      w[i] = exp(-(c[i] - lo) / lambda);
      sum += w[i];
    }
  for (int i = 0; i < K; ++i) w[i] /= sum;
}
static double clampd(double v, double lo, double hi) { return v < lo ? lo : (hi < v ? hi : v); }
void orc_update_controls(const double* nom, const double* eps, const double* w, int K, int T,
                         const double lo[2], const double hi[2], double* out) { /* :147-164 */
  for (int k = 0; k < T; ++k) {
    double dv = 0.0, dw = 0.0;
    for (int s = 0; s < K; ++s) {
      dv += w[s] * eps[((size_t)s * T + k) * 2];
      dw += w[s] * eps[((size_t)s * T + k) * 2 + 1];
    }
    out[2 * k] = clampd(nom[2 * k] + dv, lo[0], hi[0]);
    out[2 * k + 1] = clampd(nom[2 * k + 1] + dw, lo[1], hi[1]);
  }
}
void orc_shift_horizon(const double* seq, int T, double* out) { /* :166-173 */
  for (int k = 0; k + 1 < T; ++k) {
    out[2 * k] = seq[2 * (k + 1)];
    out[2 * k + 1] = seq[2 * (k + 1) + 1];
  }
  out[2 * (T - 1)] = seq[2 * (T - 1)];
  out[2 * (T - 1) + 1] = seq[2 * (T - 1) + 1];
}

struct orc_planner {
  orc_mppi_config cfg;
  int model_kind;
  const orc_gp* gp;
  int R; /* terrains */
  orc_edd5 edd5;
  double track_width;
  orc_nominal nominal;
  double p_x, chi2_2, z;
  double* nominal_seq; /* [T][2] */
  double* tw;          /* terrain weights [R] */
  double* horizon_cov; /* [T][25] */
  double* lane_r_bar;  /* [T], NULL until first tracking tick */
  double* margins;     /* [T][O] */
  int margins_O;       /* -1 until first obstacle tick */
  uint64_t tick;
  double* eps;   /* [K][T][2] */
  double* costs; /* [K] */
  double* w;     /* [K] */
  uint8_t *viol, *coll, *term, *alive;
  int threads_used;
};

int orc_planner_create(const orc_mppi_config* cfg, int kind, const orc_gp* gp, int R,
                       const orc_edd5* edd5, double track_width, const orc_nominal* nom,
                       double p_x, orc_planner** out) { /* mppi.cpp:187-202 */
  *out = NULL;
  if (!(p_x > 0.5) || !(p_x < 1.0))
    return fail(ORC_INVALID_ARGUMENT, "QuantileTables: p_x must lie in (0.5, 1)");
  if (cfg->samples < 1 || cfg->horizon < 1)
    return fail(ORC_INVALID_ARGUMENT, "MppiConfig: samples and horizon must be >= 1");
  if (!(cfg->lambda > 0.0)) return fail(ORC_INVALID_ARGUMENT, "MppiConfig: lambda must be positive");
  if (!(cfg->sigma_v2 > 0.0) || !(cfg->sigma_w2 > 0.0))
    return fail(ORC_INVALID_ARGUMENT, "MppiConfig: sampling variances must be positive");
  if (cfg->lo[0] >= cfg->hi[0] || cfg->lo[1] >= cfg->hi[1])
    return fail(ORC_INVALID_ARGUMENT, "MppiConfig: control bounds must be a nonempty box");
  if (!(nom->tau_v > 0.0) || !(nom->tau_omega > 0.0))
    return fail(ORC_INVALID_ARGUMENT, "NominalParams: time constants must be positive");
  if (!(nom->dt > 0.0) || nom->dt >= fmin(nom->tau_v, nom->tau_omega))
    return fail(ORC_INVALID_ARGUMENT, "NominalParams: require 0 < dt < min(tau_v, tau_omega)");
  if (kind == ORC_MODEL_GP && (gp == NULL || R < 1 || gp->m != 2 * R))
    return fail(ORC_INVALID_ARGUMENT, "Planner: GP ensemble needs a model with 2M outputs");
  orc_planner* p = (orc_planner*)calloc(1, sizeof(orc_planner));
  p->cfg = *cfg;
  p->model_kind = kind;
  p->gp = gp;
  p->R = kind == ORC_MODEL_GP ? R : 1;
  if (edd5) p->edd5 = *edd5;
  p->track_width = track_width;
  p->nominal = *nom;
  p->p_x = p_x;
  p->chi2_2 = orc_chi2_quantile_2dof(p_x);
  p->z = orc_normal_quantile(p_x);
  const int K = cfg->samples, T = cfg->horizon;
  p->nominal_seq = (double*)malloc(sizeof(double) * 2 * T);
  for (int k = 0; k < T; ++k) { /* bounds.clamp(Control{}) */
    p->nominal_seq[2 * k] = clampd(0.0, cfg->lo[0], cfg->hi[0]);
    p->nominal_seq[2 * k + 1] = clampd(0.0, cfg->lo[1], cfg->hi[1]);
  }
  p->tw = (double*)malloc(sizeof(double) * p->R);
  for (int i = 0; i < p->R; ++i) p->tw[i] = 1.0 / p->R;
  p->horizon_cov = (double*)calloc((size_t)T * 25, sizeof(double));
  p->margins_O = -1;
  p->eps = (double*)malloc(sizeof(double) * (size_t)K * T * 2);
  p->costs = (double*)malloc(sizeof(double) * K);
  p->w = (double*)malloc(sizeof(double) * K);
  p->viol = (uint8_t*)calloc((size_t)K * T, 1);
  p->coll = (uint8_t*)calloc((size_t)K * T, 1);
  p->term = (uint8_t*)calloc((size_t)K, 1);
  p->alive = (uint8_t*)calloc((size_t)K, 1);
  *out = p;
  return ORC_OK;
}
void orc_planner_free(orc_planner* p) {
  if (!p) return;
  free(p->nominal_seq);
  free(p->tw);
  free(p->horizon_cov);
  free(p->lane_r_bar);
  free(p->margins);
  free(p->eps);
  free(p->costs);
  free(p->w);
  free(p->viol);
  free(p->coll);
  free(p->term);
  free(p->alive);
  free(p);
}
int orc_planner_set_terrain_weights(orc_planner* p, const double* w, int R) { /* :208-218 */
  if (p->model_kind == ORC_MODEL_GP && R != p->R)
    return fail(ORC_INVALID_ARGUMENT, "set_terrain_weights: size mismatch with terrain count");
  if (!on_simplex(w, R, 1e-6))
    return fail(ORC_INVALID_ARGUMENT, "set_terrain_weights: weights must lie on the simplex");
  if (p->model_kind != ORC_MODEL_GP && R != p->R) {
    free(p->tw);
    p->tw = (double*)malloc(sizeof(double) * R);
    p->R = R;
  }
  memcpy(p->tw, w, sizeof(double) * R);
  return ORC_OK;
}

/* Per-thread rollout scratch (mppi.cpp:176-185). */
typedef struct {
  double* queries; /* cs×4 */
  double* mean;    /* cs×m */
  double* var;
  double* ws;      /* predict workspace */
  double* states;  /* cs×(T+1)×5 */
  double* trace;   /* cs×T (trace of combined covariance) */
  double* ctrl;    /* cs×T×2 */
} scratch_t;

typedef struct {
  orc_planner* p;
  const double* x0;
  const orc_task* task;
  int tid, n_threads, n_chunks;
  int use_ref_noise;
} worker_arg;

/* mppi.cpp:284-387 rollout_chunk (+ the combined-task composition) */
static void rollout_chunk(orc_planner* p, const double* x0, int lo, int hi, const orc_task* task,
                          scratch_t* sc) {
  const int cs = hi - lo, T = p->cfg.horizon;
  const int m2 = p->model_kind == ORC_MODEL_GP ? p->gp->m : 0;
  for (int i = 0; i < cs; ++i) { /* :298-308 */
    const double* e = p->eps + (size_t)(lo + i) * T * 2;
    for (int k = 0; k < T; ++k) {
      sc->ctrl[((size_t)i * T + k) * 2] = clampd(p->nominal_seq[2 * k] + e[2 * k], p->cfg.lo[0], p->cfg.hi[0]);
      sc->ctrl[((size_t)i * T + k) * 2 + 1] =
          clampd(p->nominal_seq[2 * k + 1] + e[2 * k + 1], p->cfg.lo[1], p->cfg.hi[1]);
    }
  }
  uint8_t* alive = p->alive + lo;
  for (int i = 0; i < cs; ++i) alive[i] = 1;
  memset(sc->trace, 0, sizeof(double) * (size_t)cs * T);
  if (p->model_kind == ORC_MODEL_GP) { /* :311-350 */
    const int R = p->R;
    for (int i = 0; i < cs; ++i) memcpy(sc->states + (size_t)i * (T + 1) * 5, x0, 5 * sizeof(double));
    for (int k = 0; k < T; ++k) {
      for (int i = 0; i < cs; ++i) {
        const double* s = sc->states + ((size_t)i * (T + 1) + k) * 5;
        const double* u = sc->ctrl + ((size_t)i * T + k) * 2;
        sc->queries[i * 4 + 0] = s[3];
        sc->queries[i * 4 + 1] = s[4];
        sc->queries[i * 4 + 2] = u[0];
        sc->queries[i * 4 + 3] = u[1];
      }
      predict_block(p->gp, sc->queries, cs, sc->mean, sc->var, sc->ws);
      for (int i = 0; i < cs; ++i) {
        double* s = sc->states + ((size_t)i * (T + 1) + k) * 5;
        double* nx = s + 5;
        if (!alive[i]) {
          memcpy(nx, s, 5 * sizeof(double));
          continue;
        }
        double cm[2], cv[2];
        combine(p->tw, R, sc->mean + (size_t)i * m2, sc->var + (size_t)i * m2, cm, cv);
        orc_step_nominal(s, sc->ctrl + ((size_t)i * T + k) * 2, &p->nominal, nx);
        nx[3] += cm[0];
        nx[4] += cm[1];
        if (!finite5(nx)) {
          alive[i] = 0;
          memcpy(nx, s, 5 * sizeof(double));
        }
        sc->trace[(size_t)i * T + k] = cv[0] + cv[1];
      }
    }
  } else { /* :351-368 */
    for (int i = 0; i < cs; ++i) {
      double s[5];
      memcpy(s, x0, sizeof s);
      double* st = sc->states + (size_t)i * (T + 1) * 5;
      memcpy(st, s, sizeof s);
      for (int k = 0; k < T; ++k) {
        if (alive[i]) {
          double nx[5];
          const double* u = sc->ctrl + ((size_t)i * T + k) * 2;
          if (p->model_kind == ORC_MODEL_EDD5)
            orc_step_edd5(s, u, &p->edd5, p->track_width, p->nominal.dt, nx);
          else if (p->model_kind == ORC_MODEL_UNICYCLE)
            orc_step_kinematic(s, u, p->nominal.dt, nx);
          else
            orc_step_nominal(s, u, &p->nominal, nx); /* NominalDynamic extension */
          if (!finite5(nx))
            alive[i] = 0;
          else
            memcpy(s, nx, sizeof s);
        }
        memcpy(st + 5 * (k + 1), s, sizeof s);
      }
    }
  }
  /* :370-386 costs (+ per-step flags for the parity harness) */
  const int O = task->n_obstacles;
  double* vs = (double*)malloc(sizeof(double) * T);
  for (int i = 0; i < cs; ++i) {
    const int s_idx = lo + i;
    const double* st = sc->states + (size_t)i * (T + 1) * 5;
    const double* tr = sc->trace + (size_t)i * T;
    uint8_t* viol = p->viol + (size_t)s_idx * T;
    uint8_t* coll = p->coll + (size_t)s_idx * T;
    for (int k = 0; k < T; ++k) {
      vs[k] = sc->ctrl[((size_t)i * T + k) * 2];
      const double* nx = st + 5 * (k + 1);
      viol[k] = 0;
      coll[k] = 0;
      if (task->kind != ORC_TASK_AVOIDANCE)
        viol[k] = orc_centerline_distance(task->track, nx[0], nx[1]) > p->lane_r_bar[k];
      if (task->kind != ORC_TASK_TRACKING && O > 0)
        coll[k] = orc_collision_indicator(nx[0], nx[1], task->obstacles, O,
                                          p->margins + (size_t)k * O) != 0.0;
    }
    {
      const double* last = st + 5 * T;
      const double gx = last[0] - task->goal[0], gy = last[1] - task->goal[1];
      p->term[s_idx] = task->kind == ORC_TASK_AVOIDANCE && sqrt(gx * gx + gy * gy) <= task->goal[2];
    }
    double c;
    if (!alive[i]) {
      c = NAN;
    } else if (task->kind == ORC_TASK_TRACKING) {
      c = orc_tracking_cost(st, tr, T, task->track, p->lane_r_bar, task->v_desired, vs, &task->tw);
    } else if (task->kind == ORC_TASK_AVOIDANCE) {
      c = orc_avoidance_cost(st, tr, T, task->obstacles, O, p->margins, task->goal, &task->aw,
                             task->high_cost);
    } else {
      c = orc_tracking_cost(st, tr, T, task->track, p->lane_r_bar, task->v_desired, vs, &task->tw);
      double oc = 0.0;
      for (int k = 0; k < T; ++k)
        oc += task->aw.obstacle * orc_collision_indicator(st[5 * (k + 1)], st[5 * (k + 1) + 1],
                                                          task->obstacles, O,
                                                          p->margins + (size_t)k * O);
      c += oc;
    }
    p->costs[s_idx] = c;
  }
  free(vs);
}

static void* worker(void* argp) { /* mppi.cpp:408-418 */
  worker_arg* a = (worker_arg*)argp;
  orc_planner* p = a->p;
  const int K = p->cfg.samples, T = p->cfg.horizon;
  const int n = p->model_kind == ORC_MODEL_GP ? p->gp->n : 1;
  const int m = p->model_kind == ORC_MODEL_GP ? p->gp->m : 1;
  scratch_t sc;
  sc.queries = (double*)malloc(sizeof(double) * 128 * 4);
  sc.mean = (double*)malloc(sizeof(double) * 128 * m);
  sc.var = (double*)malloc(sizeof(double) * 128 * m);
  sc.ws = (double*)malloc(sizeof(double) * 128 * 2 * (size_t)n);
  sc.states = (double*)malloc(sizeof(double) * 128 * (size_t)(T + 1) * 5);
  sc.trace = (double*)malloc(sizeof(double) * 128 * (size_t)T);
  sc.ctrl = (double*)malloc(sizeof(double) * 128 * (size_t)T * 2);
  const double sv = sqrt(p->cfg.sigma_v2), sw = sqrt(p->cfg.sigma_w2);
  for (int c = a->tid; c < a->n_chunks; c += a->n_threads) {
    const int lo = c * 128;
    const int hi = (lo + 128) < K ? (lo + 128) : K;
    if (a->use_ref_noise)
      for (int s = lo; s < hi; ++s)
        fill_perturbations(p->eps + (size_t)s * T * 2, T, sv, sw, p->cfg.seed, p->tick, (uint64_t)s);
    rollout_chunk(p, a->x0, lo, hi, a->task, &sc);
  }
  free(sc.queries);
  free(sc.mean);
  free(sc.var);
  free(sc.ws);
  free(sc.states);
  free(sc.trace);
  free(sc.ctrl);
  return NULL;
}

/* mppi.cpp:220-233 correction_at */
static void correction_at(const orc_planner* p, const double s[5], const double u[2], double cm[2],
                          double cv[2]) {
  cm[0] = cm[1] = cv[0] = cv[1] = 0.0;
  if (p->model_kind != ORC_MODEL_GP) return;
  const int m = p->gp->m;
  double q[4] = {s[3], s[4], u[0], u[1]};
  double* mean = (double*)malloc(sizeof(double) * m);
  double* var = (double*)malloc(sizeof(double) * m);
  double* ws = (double*)malloc(sizeof(double) * 2 * (size_t)p->gp->n);
  predict_block(p->gp, q, 1, mean, var, ws);
  combine(p->tw, p->R, mean, var, cm, cv);
  free(mean);
  free(var);
  free(ws);
}

/* mppi.cpp:235-282 thresholds + tightening (tracking, avoidance, or both on one chain) */
static void ensure_thresholds(orc_planner* p, const orc_task* t) {
  const int T = p->cfg.horizon;
  if (t->kind != ORC_TASK_AVOIDANCE && !p->lane_r_bar) {
    p->lane_r_bar = (double*)malloc(sizeof(double) * T);
    for (int k = 0; k < T; ++k) p->lane_r_bar[k] = t->track->half_width;
  }
  if (t->kind != ORC_TASK_TRACKING && p->margins_O != t->n_obstacles) {
    free(p->margins);
    p->margins = (double*)calloc((size_t)T * (t->n_obstacles > 0 ? t->n_obstacles : 1), sizeof(double));
    p->margins_O = t->n_obstacles;
  }
}
static void tightening_pass(orc_planner* p, const double x0[5], const orc_task* t, orc_diag* diag) {
  const int T = p->cfg.horizon, O = t->n_obstacles;
  double mu[5], cov[25];
  memcpy(mu, x0, sizeof mu);
  memset(cov, 0, sizeof cov);
  for (int k = 0; k < T; ++k) {
    const double* u = p->nominal_seq + 2 * k;
    double cm[2], cv[2], nmu[5], ncov[25];
    correction_at(p, mu, u, cm, cv);
    orc_propagate_belief(mu, cov, u, cm, cv, &p->nominal, nmu, ncov);
    memcpy(mu, nmu, sizeof mu);
    memcpy(cov, ncov, sizeof cov);
    memcpy(p->horizon_cov + (size_t)k * 25, cov, sizeof cov);
    const double cxy[4] = {cov[0], cov[1], cov[5], cov[6]};
    if (t->kind != ORC_TASK_AVOIDANCE) {
      const double r = orc_tighten_lane_radius(t->track->half_width, cxy, p->chi2_2);
      p->lane_r_bar[k] = r;
      if (r <= 0.0 && diag) diag->tightening_infeasible = 1;
    }
    if (t->kind != ORC_TASK_TRACKING) {
      for (int o = 0; o < O; ++o) {
        double d;
        const double dbar =
            orc_tighten_obstacle_distance(mu, t->obstacles + 3 * o, t->obstacles[3 * o + 2], cxy,
                                          p->z, &d, NULL, NULL);
        p->margins[(size_t)k * O + o] = d - dbar;
        if (dbar <= 0.0 && diag) diag->tightening_infeasible = 1;
      }
    }
  }
}

static int validate_track(const orc_track* t) { /* costs.cpp:44-60 */
  if (!(t->half_width > 0.0)) return fail(ORC_INVALID_ARGUMENT, "Track: half_width must be positive");
  if (t->is_circle) {
    if (!(t->radius > 0.0)) return fail(ORC_INVALID_ARGUMENT, "Track: circle radius must be positive");
    return ORC_OK;
  }
  if (t->n_waypoints < 2) return fail(ORC_INVALID_ARGUMENT, "Track: polyline needs at least 2 waypoints");
  for (int i = 1; i < t->n_waypoints; ++i) {
    const double dx = t->waypoints[2 * i] - t->waypoints[2 * i - 2];
    const double dy = t->waypoints[2 * i + 1] - t->waypoints[2 * i - 1];
    if (sqrt(dx * dx + dy * dy) < 1e-12)
      return fail(ORC_INVALID_ARGUMENT, "Track: consecutive waypoints must be distinct");
  }
  return ORC_OK;
}

static double now_ms(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec * 1e3 + ts.tv_nsec * 1e-6;
}

int orc_planner_plan_step(orc_planner* p, const double x0[5], const orc_task* task,
                          const double* eps, double command[2], orc_diag* diag) {
  const double t0 = now_ms(); /* mppi.cpp:391 */
  if (!finite5(x0)) return fail(ORC_INVALID_ARGUMENT, "plan_step: non-finite state estimate");
  if (task->kind != ORC_TASK_AVOIDANCE) {
    if (!task->track) return fail(ORC_INVALID_ARGUMENT, "plan_step: tracking task needs a track");
    int rc = validate_track(task->track);
    if (rc) return rc;
  }
  if (task->kind != ORC_TASK_TRACKING) {
    if (task->n_obstacles > 0 && !task->obstacles)
      return fail(ORC_INVALID_ARGUMENT, "plan_step: avoidance task needs an obstacle list");
  }
  if (task->kind == ORC_TASK_AVOIDANCE && !(task->high_cost > 0.0))
    return fail(ORC_INVALID_ARGUMENT, "terminal_cost: high_cost must be positive");
  ensure_thresholds(p, task);
  const int K = p->cfg.samples, T = p->cfg.horizon;
  if (eps) memcpy(p->eps, eps, sizeof(double) * (size_t)K * T * 2);
  const int n_chunks = (K + 127) / 128; /* :401-402 */
  int req = p->cfg.threads;
  if (req <= 0) {
    long hw = sysconf(_SC_NPROCESSORS_ONLN);
    req = hw > 0 ? (int)hw : 1;
  }
  const int n_threads = req < n_chunks ? req : n_chunks;
  p->threads_used = n_threads;
  worker_arg* args = (worker_arg*)malloc(sizeof(worker_arg) * n_threads);
  for (int t = 0; t < n_threads; ++t) {
    args[t].p = p;
    args[t].x0 = x0;
    args[t].task = task;
    args[t].tid = t;
    args[t].n_threads = n_threads;
    args[t].n_chunks = n_chunks;
    args[t].use_ref_noise = eps == NULL;
  }
  if (n_threads == 1) { /* :419-426 */
    worker(&args[0]);
  } else {
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * n_threads);
    for (int t = 0; t < n_threads; ++t) pthread_create(&th[t], NULL, worker, &args[t]);
    for (int t = 0; t < n_threads; ++t) pthread_join(th[t], NULL);
    free(th);
  }
  free(args);
  orc_trajectory_weights(p->costs, K, p->cfg.lambda, p->w); /* :428 */
  double* upd = (double*)malloc(sizeof(double) * 2 * T);
  orc_update_controls(p->nominal_seq, p->eps, p->w, K, T, p->cfg.lo, p->cfg.hi, upd); /* :429 */
  command[0] = upd[0]; /* :430 */
  command[1] = upd[1];
  orc_shift_horizon(upd, T, p->nominal_seq); /* :431 */
  free(upd);
  if (diag) diag->tightening_infeasible = 0; /* :432 */
  tightening_pass(p, x0, task, diag);      /* :433 */
  if (diag) { /* :435-459 */
    double best = INFINITY, sum = 0.0;
    int finite = 0;
    for (int i = 0; i < K; ++i)
      if (isfinite(p->costs[i])) {
        best = p->costs[i] < best ? p->costs[i] : best;
        sum += p->costs[i];
        ++finite;
      }
    diag->best_cost = best;
    diag->mean_cost = finite > 0 ? sum / finite : NAN;
    diag->nonfinite_samples = K - finite;
    double w2 = 0.0, h = 0.0;
    for (int i = 0; i < K; ++i) w2 += p->w[i] * p->w[i];
    diag->ess = w2 > 0.0 ? 1.0 / w2 : 0.0;
    for (int i = 0; i < K; ++i)
      if (p->w[i] > 0.0) h -= p->w[i] * log(p->w[i]);
    diag->weight_entropy = h;
    diag->plan_ms = now_ms() - t0;
  }
  ++p->tick; /* :460 */
  return ORC_OK;
}
void orc_planner_last_costs(const orc_planner* p, double* c) {
  memcpy(c, p->costs, sizeof(double) * p->cfg.samples);
}
void orc_planner_last_weights(const orc_planner* p, double* w) {
  memcpy(w, p->w, sizeof(double) * p->cfg.samples);
}
void orc_planner_last_flags(const orc_planner* p, uint8_t* viol, uint8_t* coll, uint8_t* term,
                            uint8_t* alive) {
  const size_t KT = (size_t)p->cfg.samples * p->cfg.horizon;
  if (viol) memcpy(viol, p->viol, KT);
  if (coll) memcpy(coll, p->coll, KT);
  if (term) memcpy(term, p->term, p->cfg.samples);
  if (alive) memcpy(alive, p->alive, p->cfg.samples);
}
void orc_planner_nominal_sequence(const orc_planner* p, double* s) {
  memcpy(s, p->nominal_seq, sizeof(double) * 2 * p->cfg.horizon);
}
void orc_planner_horizon_covariances(const orc_planner* p, double* c) {
  memcpy(c, p->horizon_cov, sizeof(double) * 25 * p->cfg.horizon);
}
void orc_planner_lane_radii(const orc_planner* p, double* r) {
  if (p->lane_r_bar) memcpy(r, p->lane_r_bar, sizeof(double) * p->cfg.horizon);
}
int orc_planner_obstacle_margins(const orc_planner* p, double* m) {
  if (p->margins_O <= 0) return p->margins_O < 0 ? 0 : 0;
  if (m) memcpy(m, p->margins, sizeof(double) * p->cfg.horizon * p->margins_O);
  return p->margins_O;
}
uint64_t orc_planner_tick(const orc_planner* p) { return p->tick; }
void orc_planner_set_nominal_sequence(orc_planner* p, const double* s) {
  memcpy(p->nominal_seq, s, sizeof(double) * 2 * p->cfg.horizon);
}
void orc_planner_set_thresholds(orc_planner* p, const double* r_bar, const double* margins,
                                int O) {
  const int T = p->cfg.horizon;
  if (r_bar) {
    if (!p->lane_r_bar) p->lane_r_bar = (double*)malloc(sizeof(double) * T);
    memcpy(p->lane_r_bar, r_bar, sizeof(double) * T);
  }
  if (margins) {
    free(p->margins);
    p->margins = (double*)malloc(sizeof(double) * (size_t)T * (O > 0 ? O : 1));
    memcpy(p->margins, margins, sizeof(double) * (size_t)T * O);
    p->margins_O = O;
  }
}
int orc_rollout_threads_used(const orc_planner* p) { return p->threads_used; }
