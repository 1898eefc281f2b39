/*
 * gpmppi_b200.h — C ABI of the B200-native GP-MPPI solve path.
 *
 * Drop-in boundary for the reference planner (/root/reference/proj). The
 * reference exposes a C++ class API and no FFI; each entry point below names the
 * reference interface it replaces (file:line under /root/reference/proj). Plain
 * pointers and sizes only; all host arrays are row-major FP64 unless stated.
 *
 *   state   double[5]  (x, y, theta, v, omega)              core.hpp:30-36
 *   control double[2]  (v_ref, omega_ref)                   core.hpp:54-56
 *   eps     double[K][T][2]                                 mppi.cpp:53-62 (values)
 *   kernel  double[6]  (signal_var, l0..l3, noise_var)      gp.hpp:12-22, gp.cpp:237-241
 *
 * Errors: every int-returning call returns a gpmppi_status; the message of the
 * last failure on the calling thread is gpmppi_last_error(). The codes map onto
 * the reference's exception classes (std::invalid_argument, std::runtime_error,
 * std::logic_error; SURVEY §8(b) "Error conventions"). Non-finite samples and
 * infeasible tightening are NOT errors (diag fields), as in the reference.
 *
 * There is no CPU fallback: every compute entry point runs sm_100a kernels and
 * returns GPMPPI_CUDA_ERROR when no usable device is present.
 */
#ifndef GPMPPI_B200_H
#define GPMPPI_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GPMPPI_ABI_VERSION 2

typedef enum {
  GPMPPI_OK = 0,
  GPMPPI_INVALID_ARGUMENT = 1, /* std::invalid_argument */
  GPMPPI_RUNTIME_ERROR = 2,    /* std::runtime_error (Cholesky, file IO) */
  GPMPPI_LOGIC_ERROR = 3,      /* std::logic_error */
  GPMPPI_CUDA_ERROR = 4        /* no device / launch failure */
} gpmppi_status;

const char* gpmppi_last_error(void);
int gpmppi_abi_version(void);
/* number of sm_100a kernels this library launched in this process (evidence counter) */
uint64_t gpmppi_kernel_launches(void);

/* =============================== GP model ===============================
 * Replaces gpmppi::GpModel (gp.hpp:30-98). The FP64 factorisation is computed
 * on the host exactly as gp.cpp:61-150 (kernel grouping, jitter ladder
 * 0,1e-10..1e-6, L^{-T}, alphas, LML); the device copy (Z, alpha, L^{-T} in
 * FP64 and FP32) is uploaded once and owned by the model handle. */
typedef struct gpmppi_model gpmppi_model;

/* GpModel::fit (gp.cpp:61-150). inputs n×4, outputs n×m, kernels m×6. */
int gpmppi_model_fit(const double* inputs, const double* outputs, int64_t n, int64_t m,
                     const double* kernels, int device, gpmppi_model** out);
/* GpModel::load (gp.cpp:244-272): GPMPPIG1 record, column-major FP64, refit on load. */
int gpmppi_model_load(const char* path, int device, gpmppi_model** out);
/* GpModel::save (gp.cpp:223-242): bit-exact round trip with the reference format. */
int gpmppi_model_save(const gpmppi_model* model, const char* path);
void gpmppi_model_free(gpmppi_model* model);
int gpmppi_model_n_points(const gpmppi_model* model);  /* gp.hpp:59 */
int gpmppi_model_n_outputs(const gpmppi_model* model); /* gp.hpp:60 */
int gpmppi_model_n_groups(const gpmppi_model* model);  /* gp.hpp:68 */
double gpmppi_model_group_jitter(const gpmppi_model* model, int group);       /* gp.hpp:70 */
double gpmppi_model_log_marginal_likelihood(const gpmppi_model* model, int o); /* gp.hpp:65 */
/* copies the training inputs (n×4) and outputs (n×m) back to the host */
int gpmppi_model_training_data(const gpmppi_model* model, double* inputs, double* outputs);
/* GpModel::predict_batch (gp.cpp:152-207) on the device, FP64: S×4 → mean, var S×m. */
int gpmppi_model_predict_batch(const gpmppi_model* model, const double* queries, int64_t S,
                               double* mean, double* var);
/* Per-kernel-group variance of S queries through one of the rollout variance
 * paths (GPMPPI_VAR_*; queries rounded to FP32 as in the solve): var S×G. */
int gpmppi_model_variance_batch(const gpmppi_model* model, const double* queries, int64_t S,
                                int path, double* var);

/* =============================== planner ===============================
 * Replaces gpmppi::Planner (mppi.hpp:96-143) and MppiConfig (mppi.hpp:16-26). */
typedef struct {
  int samples; /* K (MppiConfig::samples) */
  int horizon; /* T (MppiConfig::horizon) */
  double lambda;
  double sigma_v2, sigma_w2; /* MppiConfig::sigma_sim (variances) */
  double lo[2], hi[2];       /* ControlBounds (core.hpp:61-74) */
  uint64_t seed;
  int threads; /* accepted for API parity; results never depend on it */
} gpmppi_mppi_config;

typedef struct {
  double tau_v, tau_omega, dt; /* NominalParams (dynamics.hpp:12-18) */
} gpmppi_nominal;

typedef struct {
  double alpha_l, alpha_r, x_icr, y_icr_l, y_icr_r; /* Edd5Params (dynamics.hpp:36-45) */
} gpmppi_edd5;

enum {
  GPMPPI_MODEL_GP_ENSEMBLE = 0, /* GpEnsemble (mppi.hpp:30-33) */
  GPMPPI_MODEL_EDD5 = 1,        /* Edd5Baseline (mppi.hpp:34-37) */
  GPMPPI_MODEL_UNICYCLE = 2,    /* UnicycleBaseline (mppi.hpp:38) */
  GPMPPI_MODEL_NOMINAL = 3      /* extension: dynamic unicycle, zero residual (BASELINE config 1) */
};

typedef struct {
  int kind;
  const gpmppi_model* gp; /* non-owning, as GpEnsemble::model (mppi.hpp:31) */
  int n_terrains;
  gpmppi_edd5 edd5;
  double track_width;
} gpmppi_prediction_model;

/* Models file GPMPPIM1 (harness.cpp:249-284): magic, EDD5 params (5 f64),
 * nominal (3 f64), has_gp byte, then a GPMPPIG1 record. gp is NULL when the file
 * carries no GP. */
int gpmppi_models_load(const char* path, int device, gpmppi_edd5* edd5, gpmppi_nominal* nominal,
                       gpmppi_model** gp);
int gpmppi_models_save(const char* path, const gpmppi_edd5* edd5, const gpmppi_nominal* nominal,
                       const gpmppi_model* gp);

typedef struct { /* Track (costs.hpp:13-27) */
  int is_circle;
  double cx, cy, radius;
  int n_waypoints;         /* <= GPMPPI_MAX_WAYPOINTS */
  const double* waypoints; /* [W][2] */
  int closed;
  double half_width;
} gpmppi_track;

typedef struct {
  double variance, deviation, slip, safety, speed; /* TrackingWeights (costs.hpp:34-40) */
} gpmppi_tracking_weights;

typedef struct {
  double variance, obstacle, stage, terminal; /* AvoidanceWeights (costs.hpp:44-50) */
} gpmppi_avoidance_weights;

enum {
  GPMPPI_TASK_TRACKING = 0,  /* TrackingTask  (mppi.hpp:42-46) */
  GPMPPI_TASK_AVOIDANCE = 1, /* AvoidanceTask (mppi.hpp:47-52) */
  GPMPPI_TASK_COMBINED = 2   /* tracking_cost + obstacle·Σ collision */
};
#define GPMPPI_MAX_WAYPOINTS 64
#define GPMPPI_MAX_OBSTACLES 64

typedef struct {
  int kind;
  const gpmppi_track* track; /* tracking / combined */
  double v_desired;
  gpmppi_tracking_weights tracking;
  const double* obstacles; /* [O][3] (cx, cy, r); avoidance / combined */
  int n_obstacles;
  double goal[3]; /* (x, y, capture_radius) GoalSpec (costs.hpp:52-55) */
  gpmppi_avoidance_weights avoidance;
  double high_cost; /* AvoidanceTask::high_cost (mppi.hpp:51) */
} gpmppi_task;

typedef struct { /* StepDiagnostics (mppi.hpp:81-89) */
  double best_cost, mean_cost, ess, weight_entropy;
  int nonfinite_samples;
  int tightening_infeasible;
  double plan_ms;    /* host wall clock of the whole call (as mppi.cpp:456-458) */
  double command_ms; /* host wall clock until the command was available */
} gpmppi_diag;

typedef struct gpmppi_planner gpmppi_planner;

/* Planner(cfg, model, nominal, p_x) (mppi.cpp:187-202) */
int gpmppi_planner_create(const gpmppi_mppi_config* cfg, const gpmppi_prediction_model* model,
                          const gpmppi_nominal* nominal, double p_x, int device,
                          gpmppi_planner** out);
void gpmppi_planner_free(gpmppi_planner* p);
/* B independent planners sharing one model (BASELINE config 4):
 * robot b behaves exactly like gpmppi_planner_create with cfg.seed = seeds[b]
 * (seeds may be NULL: cfg.seed + b). Every per-robot array of the getters/setters
 * below is robot-major ([B][...]); B = 1 gives the single-planner layout. */
int gpmppi_planner_create_batch(const gpmppi_mppi_config* cfg, const gpmppi_prediction_model* model,
                                const gpmppi_nominal* nominal, double p_x, int n_robots,
                                const uint64_t* seeds, int device, gpmppi_planner** out);
int gpmppi_planner_robots(const gpmppi_planner* p);
/* Planner::plan_step (mppi.cpp:389-475), both overloads + the combined task. Host
 * buffers in, host command out; the GPU work runs on the planner's stream. */
int gpmppi_planner_plan_step(gpmppi_planner* p, const double x0[5], const gpmppi_task* task,
                             double command[2], gpmppi_diag* diag);
/* one tick of every robot: x0 [B][5], tasks [B], commands [B][2], diags [B] or NULL */
int gpmppi_planner_plan_step_batch(gpmppi_planner* p, const double* x0, const gpmppi_task* tasks,
                                   double* commands, gpmppi_diag* diags);
/* Planner::set_terrain_weights (mppi.cpp:208-218): every robot / one robot */
int gpmppi_planner_set_terrain_weights(gpmppi_planner* p, const double* w, int R);
int gpmppi_planner_set_robot_terrain_weights(gpmppi_planner* p, int robot, const double* w, int R);
int gpmppi_planner_terrain_weights(const gpmppi_planner* p, double* w);      /* [B][R], returns R */
int gpmppi_planner_nominal_sequence(const gpmppi_planner* p, double* seq);   /* [B][T][2] */
int gpmppi_planner_set_nominal_sequence(gpmppi_planner* p, const double* seq);
int gpmppi_planner_horizon_covariances(const gpmppi_planner* p, double* cov); /* [B][T][5][5] */
int gpmppi_planner_lane_radii(const gpmppi_planner* p, double* r);    /* [B][T]; returns T, 0 if no robot has radii yet */
/* [B][T][O] with O = max obstacle count over robots (zero-padded); returns O */
int gpmppi_planner_obstacle_margins(const gpmppi_planner* p, double* m);
int gpmppi_planner_set_thresholds(gpmppi_planner* p, const double* r_bar, const double* margins,
                                  int n_obstacles); /* [B][T], [B][T][n_obstacles] */
uint64_t gpmppi_planner_tick(const gpmppi_planner* p);
int gpmppi_planner_horizon(const gpmppi_planner* p);
int gpmppi_planner_samples(const gpmppi_planner* p);

/* ---- noise (north star: Philox production sampler + injection hook) ---- */
enum { GPMPPI_NOISE_PHILOX = 0, GPMPPI_NOISE_INJECTED = 1 };
int gpmppi_planner_set_noise_mode(gpmppi_planner* p, int mode);
/* eps [B][K][T][2] (this rank's samples), used by every following tick until replaced */
int gpmppi_planner_inject_noise(gpmppi_planner* p, const double* eps);
/* materialise the Philox noise the planner uses at tick t ([B][K][T][2]) */
int gpmppi_planner_philox_noise(const gpmppi_planner* p, uint64_t tick, double* eps);

/* ---- parity outputs of the last plan_step ---- */
int gpmppi_planner_sample_costs(const gpmppi_planner* p, double* costs);   /* [B][K] */
int gpmppi_planner_sample_weights(const gpmppi_planner* p, double* w);     /* [B][K] */
/* per-step lane-violation and collision flags [B][K][T], terminal-capture and alive [B][K] */
int gpmppi_planner_flags(const gpmppi_planner* p, uint8_t* viol, uint8_t* coll,
                         uint8_t* terminal, uint8_t* alive);

/* ---- variance path (north star: tensor cores only where tolerance allows) ----
 * FFMA: FP32 CUDA cores. TC_3XTF32: tcgen05 kind::tf32, hi/lo splits, three products.
 * TC_1XTF32: one TF32 product (not a parity path). TC_3XF16 (default): tcgen05 kind::f16
 * on scaled hi/lo FP16 operands -- the same 22-bit splits at twice the TF32 rate; the
 * library runs it on single CTAs or CTA pairs by shape.
 * TC_3XF16_PAIR forces the CTA-pair kernel. Measured bounds: tests/test_gpu_variance_paths.py. */
enum {
  GPMPPI_VAR_FFMA = 0,
  GPMPPI_VAR_TC_3XTF32 = 1,
  GPMPPI_VAR_TC_1XTF32 = 2,
  GPMPPI_VAR_TC_3XF16 = 3,
  GPMPPI_VAR_TC_3XF16_PAIR = 4 /* CTA pairs (tcgen05 cta_group::2, M = 256) */
};
int gpmppi_planner_set_variance_path(gpmppi_planner* p, int path);
int gpmppi_planner_variance_path(const gpmppi_planner* p);

/* ---- device-resident timing (bench): run `ticks` plan steps back to back on
 * device-resident inputs (x0 held fixed). tick_ms[t] = CUDA-event time of tick t
 * on the planner's stream; with flush_l2 a >L2-sized memset runs between ticks
 * outside the timed spans. phase_ms[0..3] = summed event time of rollout,
 * variance, reduce+update, tightening. */
int gpmppi_planner_bench_device(gpmppi_planner* p, const double* x0, const gpmppi_task* tasks,
                                int ticks, int flush_l2, double* tick_ms, double* phase_ms);
/* write a buffer twice the L2 size on `device` and synchronise */
int gpmppi_flush_l2(int device);
/* bytes one plan_step copies host->device (robot tick blocks + tasks) and device->host
 * (command + diag), all robots */
int gpmppi_planner_io_bytes(const gpmppi_planner* p, int64_t* h2d, int64_t* d2h);

/* ---- sharded solve (multi-GPU) ----
 * A planner can own a contiguous global sample range [begin, begin+count) of a
 * solve with cfg.samples = total; noise is keyed by the GLOBAL sample index.
 * plan_partial writes this rank's reduction tuple (gpmppi_tuple_doubles(T)
 * doubles) to a DEVICE buffer; the caller all-gathers the tuples (NCCL) and
 * plan_finish combines them in rank order, updates/shifts the sequence, runs
 * the tightening pass and returns the command. */
/* diagnostics: per-role cycle counters of the tensor-core variance kernel,
 * filled when GPMPPI_TC_DEBUG has bit 512 set; read-and-reset */
int gpmppi_debug_tc_profile(double* out16);
/* diagnostics: clock64 timeline of CTA 0 of the last tensor-core variance launch
 * (GPMPPI_TC_DEBUG bit 4096): entry, role tile starts, accumulator hand-offs */
int gpmppi_debug_tc_trace(double* out64);
/* diagnostics: %globaltimer stamps (ns) at fixed points of the last tick, filled by a
 * -DGPM_TIMELINE build (tools/timeline.py); zeros otherwise; read-and-reset */
int gpmppi_debug_timeline(double* out32);
int gpmppi_tuple_doubles(int horizon);
int gpmppi_planner_set_shard(gpmppi_planner* p, int64_t begin, int64_t count);
int gpmppi_planner_plan_partial(gpmppi_planner* p, const double x0[5], const gpmppi_task* task,
                                void* device_tuple_out);
int gpmppi_planner_plan_finish(gpmppi_planner* p, const void* device_tuples, int n_ranks,
                               double command[2], gpmppi_diag* diag);
/* In-library NCCL exchange (replaces the reference's single exchange point, the
 * softmax reduction of mppi.cpp:428-429, for a solve sharded over GPUs):
 * gpmppi_nccl_unique_id fills a 128-byte ncclUniqueId on one rank (the caller
 * broadcasts it); every rank then calls gpmppi_planner_attach_comm (collective), which
 * takes the rank's contiguous global sample range of cfg.samples. From then on
 * gpmppi_planner_plan_step runs the sharded tick on the planner stream: rollout ->
 * variance -> reduce -> ncclAllGather of the (2T+6)-double tuples -> rank-order combine
 * + update + shift (identical on every rank) -> command -> tightening. No host sync
 * inside the tick; it is captured in the tick's CUDA graph like the single-GPU tick. */
int gpmppi_nccl_unique_id(void* out128);
int gpmppi_planner_attach_comm(gpmppi_planner* p, const void* unique_id, int n_ranks, int rank);
int gpmppi_planner_shard(const gpmppi_planner* p, int64_t* begin, int64_t* count, int* n_ranks,
                         int* rank);
/* Command-first mode (default off = reference semantics): plan_step returns as soon as the
 * command and the sample diagnostics are on the host; the tightening pass, which only the
 * next tick consumes (mppi.cpp:235-248), completes behind the return. Its outputs are
 * waited for by the next plan_step, by every accessor, and by wait_tightening, which also
 * completes that tick's diag (tightening_infeasible; plan_ms = launch latency + device
 * span of the whole tick). diag.command_ms is the time to command in both modes. */
int gpmppi_planner_set_command_first(gpmppi_planner* p, int on);
int gpmppi_planner_wait_tightening(gpmppi_planner* p, gpmppi_diag* diag);
/* Host restatement of the tuple combine the device runs (for CPU multi-rank tests):
 * tuples n_ranks×gpmppi_tuple_doubles(T) → combined tuple. */
int gpmppi_combine_tuples_host(const double* tuples, int n_ranks, int horizon, double lambda,
                               double* out);

/* ---- reference free functions (mppi.hpp:60-79), computed on `device` ----
 * Host buffers in and out; each call synchronises. */
/* rollout (mppi.cpp:80-111): mean-only rollout of one sequence seq[T][2];
 * states[(T+1)][5], corrections[T][4] = (mean_v, mean_w, var_v, var_w) (GaussianCorrection) */
int gpmppi_rollout(const gpmppi_prediction_model* model, const gpmppi_nominal* nominal,
                   const double* terrain_weights, int R, const double x0[5], const double* seq, int T,
                   int device, double* states, double* corrections);
/* sample_perturbations (mppi.cpp:113-123) with the production Philox sampler: eps[K][T][2] */
int gpmppi_sample_perturbations(const gpmppi_mppi_config* cfg, uint64_t tick, int device, double* eps);
/* trajectory_weights (mppi.cpp:125-145) */
int gpmppi_trajectory_weights(const double* costs, int64_t K, double lambda, int device, double* w);
/* update_controls (mppi.cpp:147-164): nominal[T][2], eps[K][T][2], w[K] -> out[T][2] */
int gpmppi_update_controls(const double* nominal, int T, const double* eps, const double* w, int64_t K,
                           const double lo[2], const double hi[2], int device, double* out);
/* shift_horizon (mppi.cpp:166-173) */
int gpmppi_shift_horizon(const double* seq, int T, int device, double* out);

/* select_kernel_grid (gp.cpp:274-366): shared-kernel hyperparameters by the reference's
 * coarse 5x7x5 LML grid plus one 5x7x5 refinement; every cell's Cholesky and LML on the
 * device. inputs n x 4, outputs n x m row-major; kernel6 = (sv, l0..l3, nv) of the winner,
 * best_lml (optional) its summed log marginal likelihood. */
int gpmppi_select_kernel_grid(const double* inputs, const double* outputs, int64_t n, int64_t m, int device,
                              double kernel6[6], double* best_lml);

/* ---- the reference's scalar helpers (bindings/module.cpp:40-181), host C++ ----
 * Same arithmetic as the planner's kernels (common.cuh); return GPMPPI_INVALID_ARGUMENT
 * with the reference's message where the reference throws std::invalid_argument. */
double gpmppi_wrap_angle(double angle);                                               /* core.hpp:18-27 */
int gpmppi_step_nominal(const double s[5], const double u[2], const gpmppi_nominal* p, double out[5]);
int gpmppi_step_kinematic_unicycle(const double s[5], const double u[2], double dt, double out[5]);
int gpmppi_step_edd5(const double s[5], const double u[2], const gpmppi_edd5* p, double track_width, double dt,
                     double out[5]);                                                   /* dynamics.cpp:59-127 */
int gpmppi_jacobian_nominal(const double s[5], const double u[2], const gpmppi_nominal* p,
                            double J[25]);                                             /* dynamics.cpp:68-98, row-major */
int gpmppi_body_frame_displacement(const double from[5], const double to[5], double out[2]); /* core.hpp:117-126 */
int gpmppi_kernel_eval(const double a[4], const double b[4], const double kernel6[6], double* out); /* gp.cpp:53-60 */
/* gp.cpp:368-389: means / var_diags m x 2 row-major, weights m on the simplex (1e-6) */
int gpmppi_ensemble_combine(const double* means, const double* var_diags, const double* weights, int m,
                            double mean[2], double cov[4]);
int gpmppi_project_simplex(const double* z, int m, double* out);                       /* terrain.cpp:72-92 */
int gpmppi_chi2_quantile_2dof(double p, double* out);                                   /* uncertainty.cpp:8-13 */
int gpmppi_normal_quantile(double p, double* out);                                      /* uncertainty.cpp:54-60 */
double gpmppi_normal_cdf(double x);                                                     /* uncertainty.cpp:15 */
int gpmppi_tighten_lane_radius(double r, const double cov_xy[4], double p_x, double* out); /* :90-96 */
int gpmppi_tighten_obstacle_distance(const double robot_xy[2], const double center[2], double radius,
                                     const double cov_xy[4], double p_x, double* d_bar, double normal[2],
                                     int* degenerate, double* d);                        /* :98-116 */

#ifdef __cplusplus
}
#endif
#endif
