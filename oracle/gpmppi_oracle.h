/*
 * gpmppi_oracle.h — CPU (FP64) restatement of the reference GP-MPPI solve path.
 *
 * TEST INFRASTRUCTURE ONLY. This is the parity checker and the CPU baseline
 * ("port" kind) — it is never linked into, called by, or shipped with the
 * product library (paper_2411_03289_b200/lib/libgpmppi_b200.so). Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load it.
 *
 * Every function cites the reference file:line it restates (paths relative to
 * /root/reference/proj). The reference itself cannot be built here (Eigen3,
 * doctest, CLI11 and the vendored json.hpp are absent), so the restatement is
 * pinned by (1) the reference's own inline known-answer tests, ported to
 * tests/test_oracle_kat.py, and (2) the reference's Eigen-free RNG header
 * compiled from the read-only tree by oracle/build_ref.sh into oracle/_ref/.
 *
 * Layout conventions (shared with the C-ABI in include/gpmppi_b200.h):
 *   state   double[5]  = (x, y, theta, v, omega)          core.hpp:30-36
 *   control double[2]  = (v_ref, omega_ref)                core.hpp:54-56
 *   eps     double[K][T][2]  (sample-major, then step, then channel)
 *   GP inputs double[n][4], outputs double[n][m] (row-major)
 *   kernel  double[6]  = (signal_var, l0, l1, l2, l3, noise_var)  gp.cpp:237-241
 */
#ifndef GPMPPI_ORACLE_H
#define GPMPPI_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status (mirrors the reference's exception classes) ---- */
enum { ORC_OK = 0, ORC_INVALID_ARGUMENT = 1, ORC_RUNTIME_ERROR = 2, ORC_LOGIC_ERROR = 3 };
const char* orc_last_error(void);

/* ---- rng.hpp:11-68 ---- */
uint64_t orc_splitmix64(uint64_t x);
uint64_t orc_derive_seed(uint64_t seed, uint64_t a, uint64_t b);
typedef struct {
  uint64_t mt[312];
  int mti;
  int has_spare;
  double spare;
} orc_rng;
void orc_rng_seed(orc_rng* r, uint64_t seed);
uint64_t orc_rng_next(orc_rng* r);
double orc_rng_uniform01(orc_rng* r);
double orc_rng_uniform(orc_rng* r, double lo, double hi);
void orc_rng_gaussian_pair(orc_rng* r, double* z1, double* z2);
double orc_rng_gaussian(orc_rng* r);
void orc_uniform_stream(uint64_t seed, int n, double* out);
void orc_gaussian_stream(uint64_t seed, int n, double* out);
/* mppi.cpp:113-123 — eps[K][T][2] for (seed, tick). sigma_sim are variances. */
void orc_sample_perturbations(int K, int T, double sigma_v2, double sigma_w2, uint64_t seed,
                              uint64_t tick, double* eps);

/* ---- core.hpp / dynamics.cpp ---- */
typedef struct {
  double tau_v, tau_omega, dt;
} orc_nominal;
typedef struct {
  double alpha_l, alpha_r, x_icr, y_icr_l, y_icr_r;
} orc_edd5;
double orc_wrap_angle(double a);
void orc_arc_advance(double* x, double* y, double* th, double vx, double vy, double om, double dt);
void orc_step_nominal(const double s[5], const double u[2], const orc_nominal* p, double out[5]);
void orc_jacobian_nominal(const double s[5], const double u[2], const orc_nominal* p,
                          double J[25]);
void orc_step_kinematic(const double s[5], const double u[2], double dt, double out[5]);
void orc_step_edd5(const double s[5], const double u[2], const orc_edd5* p, double track_width,
                   double dt, double out[5]);

/* ---- gp.cpp ---- */
typedef struct orc_gp orc_gp;
int orc_gp_fit(const double* inputs, const double* outputs, int n, int m, const double* kernels,
               orc_gp** out);
void orc_gp_free(orc_gp* g);
int orc_gp_n_points(const orc_gp* g);
int orc_gp_n_outputs(const orc_gp* g);
int orc_gp_n_groups(const orc_gp* g);
double orc_gp_group_jitter(const orc_gp* g, int grp);
double orc_gp_lml(const orc_gp* g, int output);
/* copies (L^{-T}) n×n row-major, alphas n×|outputs| row-major, inputs_aug n×6 */
void orc_gp_group_export(const orc_gp* g, int grp, double* inv_lower_t, double* chol_lower,
                         double* alphas, double* inputs_aug, int* outputs, int* n_outputs,
                         double* kernel6);
int orc_gp_predict_batch(const orc_gp* g, const double* queries, int S, double* mean,
                         double* var);
double orc_kernel_eval(const double a[4], const double b[4], const double kernel6[6]);
/* gp.cpp:368-389; means/vars [R][2], w[R] → mean[2], cov_diag[2] */
int orc_ensemble_combine(const double* means, const double* vars, const double* w, int R,
                         double mean[2], double cov_diag[2]);

/* ---- uncertainty.cpp ---- */
double orc_chi2_quantile_2dof(double p);
double orc_normal_cdf(double x);
double orc_normal_quantile(double p);
double orc_lambda_max_2x2(const double m[4]);
void orc_propagate_belief(const double mean[5], const double cov[25], const double u[2],
                          const double corr_mean[2], const double corr_cov_diag[2],
                          const orc_nominal* p, double out_mean[5], double out_cov[25]);
double orc_tighten_lane_radius(double r, const double cov_xy[4], double chi2_2);
double orc_tighten_obstacle_distance(const double xy[2], const double c[2], double radius,
                                     const double cov_xy[4], double z, double* d_out,
                                     double normal[2], int* degenerate);

/* ---- costs.cpp ---- */
typedef struct {
  int is_circle;
  double cx, cy, radius;
  int n_waypoints;
  const double* waypoints; /* [W][2] */
  int closed;
  double half_width;
} orc_track;
typedef struct {
  double variance, deviation, slip, safety, speed;
} orc_tracking_weights;
typedef struct {
  double variance, obstacle, stage, terminal;
} orc_avoidance_weights;
double orc_centerline_distance(const orc_track* t, double x, double y);
double orc_slip_ratio(const double prev[5], const double next[5]);
double orc_collision_indicator(double x, double y, const double* obstacles, int O,
                               const double* margins);
/* states [N+1][5], corr_trace [N] (trace of combined covariance), r_bar [N], v_sampled [N] */
double orc_tracking_cost(const double* states, const double* corr_trace, int N,
                         const orc_track* track, const double* r_bar, double v_desired,
                         const double* v_sampled, const orc_tracking_weights* w);
double orc_avoidance_cost(const double* states, const double* corr_trace, int N,
                          const double* obstacles, int O, const double* margins,
                          const double goal[3], const orc_avoidance_weights* w,
                          double high_cost);

/* ---- mppi.cpp ---- */
void orc_trajectory_weights(const double* costs, int K, double lambda, double* w);
void orc_update_controls(const double* nominal, const double* eps, const double* w, int K,
                         int T, const double lo[2], const double hi[2], double* out);
void orc_shift_horizon(const double* seq, int T, double* out);
/* mppi.cpp:80-111 rollout (mean-only, one sequence): states (T+1)x5, corr Tx4 */
int orc_rollout(int kind, const orc_gp* gp, int R, const double* w, const orc_nominal* nom,
                const orc_edd5* edd, double track_width, const double x0[5], const double* seq,
                int T, double* states, double* corr);

enum { ORC_MODEL_GP = 0, ORC_MODEL_EDD5 = 1, ORC_MODEL_UNICYCLE = 2, ORC_MODEL_NOMINAL = 3 };
enum { ORC_TASK_TRACKING = 0, ORC_TASK_AVOIDANCE = 1, ORC_TASK_COMBINED = 2 };

typedef struct {
  int samples, horizon;
  double lambda;
  double sigma_v2, sigma_w2; /* sampling variances (MppiConfig::sigma_sim) */
  double lo[2], hi[2];       /* ControlBounds */
  uint64_t seed;
  int threads;
} orc_mppi_config;

typedef struct {
  int kind; /* ORC_TASK_* */
  /* tracking (and combined) */
  const orc_track* track;
  double v_desired;
  orc_tracking_weights tw;
  /* avoidance (and combined obstacle term) */
  const double* obstacles; /* [O][3] */
  int n_obstacles;
  double goal[3]; /* px, py, capture_radius */
  orc_avoidance_weights aw;
  double high_cost;
} orc_task;

typedef struct {
  double best_cost, mean_cost, ess, weight_entropy;
  int nonfinite_samples;
  int tightening_infeasible;
  double plan_ms;
} orc_diag;

typedef struct orc_planner orc_planner;
int orc_planner_create(const orc_mppi_config* cfg, int model_kind, const orc_gp* gp,
                       int n_terrains, const orc_edd5* edd5, double track_width,
                       const orc_nominal* nominal, double p_x, orc_planner** out);
void orc_planner_free(orc_planner* p);
int orc_planner_set_terrain_weights(orc_planner* p, const double* w, int R);
/* eps == NULL → reference mt19937_64 noise (mppi.cpp:408-415); else injected [K][T][2] */
int orc_planner_plan_step(orc_planner* p, const double x0[5], const orc_task* task,
                          const double* eps, double command[2], orc_diag* diag);
/* parity outputs of the last plan_step */
void orc_planner_last_costs(const orc_planner* p, double* costs);   /* [K] */
void orc_planner_last_weights(const orc_planner* p, double* w);     /* [K] */
void orc_planner_last_flags(const orc_planner* p, uint8_t* viol, uint8_t* coll,
                            uint8_t* terminal_hit, uint8_t* alive); /* [K][T],[K][T],[K],[K] */
void orc_planner_nominal_sequence(const orc_planner* p, double* seq); /* [T][2] */
void orc_planner_horizon_covariances(const orc_planner* p, double* cov); /* [T][25] */
void orc_planner_lane_radii(const orc_planner* p, double* r);           /* [T] */
int orc_planner_obstacle_margins(const orc_planner* p, double* m);     /* [T][O], returns O */
uint64_t orc_planner_tick(const orc_planner* p);
void orc_planner_set_nominal_sequence(orc_planner* p, const double* seq);
/* replace thresholds (for parity runs that start mid-trajectory) */
void orc_planner_set_thresholds(orc_planner* p, const double* r_bar, const double* margins,
                                int O);
int orc_rollout_threads_used(const orc_planner* p);
/* Timed CPU baseline only: route gp.cpp's GEMM / GEMM / TRMM through a dlopen'd CBLAS
 * (symbol prefix e.g. "scipy_"); NULL path restores the scalar checker loops. */
int orc_use_blas(const char* so_path, const char* prefix);

#ifdef __cplusplus
}
#endif
#endif
