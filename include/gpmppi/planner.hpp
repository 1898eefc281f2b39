// gpmppi/planner.hpp — header-only C++ drop-in for the reference planner API
// (/root/reference/proj/include/gpmppi/{mppi,gp,costs,dynamics,core}.hpp) on top
// of the C ABI in gpmppi_b200.h. Same class / member names, argument meaning and
// exception types (std::invalid_argument, std::runtime_error, std::logic_error).
//
// Eigen is not a dependency. The value types here (Vec<N>, Vector, Matrix, Mat<R,C>)
// give the element access the reference's callers use -- v(i), m(i, j), rows(),
// cols(), size() -- and every entry point that takes an Eigen type in the reference
// is a template accepting any type with that interface, so Eigen::Vector2d /
// Vector4d / VectorXd / MatrixXd / MatrixX2d arguments work unchanged:
//   GpModel::fit(inputs n×4, outputs n×m, kernels)          gp.hpp:34-35
//   GpModel::predict(q), predict_batch(Q), predict_batch_into(Q, mean, var, ws)  gp.hpp:41-57
//   Track::circle_track(center, r, hw), polyline_track(pts, hw, closed)          costs.hpp:21-22
//   MppiConfig::sigma_sim(i), KernelParams::lengthscales(i)                      mppi.hpp:20, gp.hpp:14
//   rollout / sample_perturbations / trajectory_weights / update_controls        mppi.hpp:60-79
//   Planner::set_terrain_weights(TerrainWeights{w}), RobotState::from_vec(v)     mppi.hpp:108, core.hpp:46
// Link with -lgpmppi_b200 (paper_2411_03289_b200/lib/libgpmppi_b200.so).
#pragma once

#include <array>
#include <cstdint>
#include <initializer_list>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <variant>
#include <vector>

#include "gpmppi_b200.h"

namespace gpmppi {

namespace detail {
inline void check(int rc) {
  if (rc == GPMPPI_OK) return;
  const std::string msg = gpmppi_last_error();
  switch (rc) {
    case GPMPPI_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case GPMPPI_LOGIC_ERROR: throw std::logic_error(msg);
    default: throw std::runtime_error(msg);  // runtime errors and CUDA failures
  }
}
// element access of the caller's vector / matrix types: v(i) (Eigen) or v[i] (std containers)
template <class V, class = void>
struct has_call1 : std::false_type {};
template <class V>
struct has_call1<V, std::void_t<decltype(std::declval<const V&>()(0))>> : std::true_type {};
template <class M, class = void>
struct is_matrix : std::false_type {};
template <class M>
struct is_matrix<M, std::void_t<decltype(std::declval<const M&>()(0, 0)), decltype(std::declval<const M&>().rows()),
                                decltype(std::declval<const M&>().cols())>> : std::true_type {};
template <class V>
double at(const V& v, long i) {
  if constexpr (has_call1<V>::value)
    return static_cast<double>(v(i));
  else
    return static_cast<double>(v[i]);
}
template <class V>
long length(const V& v) {
  return static_cast<long>(v.size());
}
}  // namespace detail

// Fixed-size vector (Eigen::Vector2d / Vector4d / Vector5d stand-in).
template <int N>
struct Vec {
  double v[N]{};
  Vec() = default;
  template <class... T, class = std::enable_if_t<sizeof...(T) == N && (std::is_arithmetic_v<T> && ...)>>
  Vec(T... x) : v{static_cast<double>(x)...} {}
  template <class O, class = std::enable_if_t<!std::is_arithmetic_v<O> && !std::is_same_v<std::decay_t<O>, Vec> &&
                                              (detail::has_call1<O>::value || detail::is_matrix<O>::value)>>
  Vec(const O& o) {  // from any vector with v(i) (e.g. an Eigen fixed-size vector)
    for (int i = 0; i < N; ++i) v[i] = detail::at(o, i);
  }
  double& operator()(long i) { return v[i]; }
  double operator()(long i) const { return v[i]; }
  double& operator[](long i) { return v[i]; }
  double operator[](long i) const { return v[i]; }
  static constexpr long size() { return N; }
  static constexpr long rows() { return N; }
  static constexpr long cols() { return 1; }
  double* data() { return v; }
  const double* data() const { return v; }
  double* begin() { return v; }
  double* end() { return v + N; }
  const double* begin() const { return v; }
  const double* end() const { return v + N; }
};
using Vec2 = Vec<2>;
using Vec4 = Vec<4>;
using Vec5 = Vec<5>;

// Dynamic vector (Eigen::VectorXd stand-in).
class Vector {
 public:
  Vector() = default;
  explicit Vector(long n, double fill = 0.0) : d_(static_cast<size_t>(n), fill) {}
  Vector(std::initializer_list<double> l) : d_(l) {}
  explicit Vector(std::vector<double> d) : d_(std::move(d)) {}
  template <class O, class = std::enable_if_t<!std::is_arithmetic_v<O> && detail::has_call1<O>::value &&
                                              !std::is_same_v<std::decay_t<O>, Vector>>>
  Vector(const O& o) : d_(static_cast<size_t>(o.size())) {
    for (long i = 0; i < size(); ++i) d_[i] = detail::at(o, i);
  }
  static Vector Constant(long n, double x) { return Vector(n, x); }
  double& operator()(long i) { return d_[i]; }
  double operator()(long i) const { return d_[i]; }
  double& operator[](long i) { return d_[i]; }
  double operator[](long i) const { return d_[i]; }
  long size() const { return static_cast<long>(d_.size()); }
  long rows() const { return size(); }
  static constexpr long cols() { return 1; }
  void resize(long n) { d_.resize(static_cast<size_t>(n)); }
  double* data() { return d_.data(); }
  const double* data() const { return d_.data(); }
  auto begin() { return d_.begin(); }
  auto end() { return d_.end(); }
  auto begin() const { return d_.begin(); }
  auto end() const { return d_.end(); }
  const std::vector<double>& std() const { return d_; }

 private:
  std::vector<double> d_;
};

// Dynamic matrix, row-major storage (Eigen::MatrixXd / MatrixX2d stand-in).
class Matrix {
 public:
  Matrix() = default;
  Matrix(long r, long c, double fill = 0.0) : r_(r), c_(c), d_(static_cast<size_t>(r * c), fill) {}
  template <class O, class = std::enable_if_t<detail::is_matrix<O>::value && !std::is_same_v<std::decay_t<O>, Matrix>>>
  Matrix(const O& o) : Matrix(static_cast<long>(o.rows()), static_cast<long>(o.cols())) {
    for (long i = 0; i < r_; ++i)
      for (long j = 0; j < c_; ++j) (*this)(i, j) = static_cast<double>(o(i, j));
  }
  double& operator()(long i, long j) { return d_[static_cast<size_t>(i * c_ + j)]; }
  double operator()(long i, long j) const { return d_[static_cast<size_t>(i * c_ + j)]; }
  long rows() const { return r_; }
  long cols() const { return c_; }
  long size() const { return r_ * c_; }
  void resize(long r, long c) {
    r_ = r;
    c_ = c;
    d_.assign(static_cast<size_t>(r * c), 0.0);
  }
  double* data() { return d_.data(); }  // row-major
  const double* data() const { return d_.data(); }

 private:
  long r_ = 0, c_ = 0;
  std::vector<double> d_;
};

// Fixed-size matrix (Eigen::Matrix2d / Matrix5d stand-in), row-major.
template <int R, int C>
struct Mat {
  double m[R * C]{};
  double& operator()(long i, long j) { return m[i * C + j]; }
  double operator()(long i, long j) const { return m[i * C + j]; }
  static constexpr long rows() { return R; }
  static constexpr long cols() { return C; }
  double* data() { return m; }
  const double* data() const { return m; }
};
using Matrix2d = Mat<2, 2>;
using Matrix5d = Mat<5, 5>;

struct RobotState {  // core.hpp:30-51
  double x{0.0}, y{0.0}, theta{0.0}, v{0.0}, omega{0.0};
  Vec5 vec() const { return {x, y, theta, v, omega}; }
  template <class V>
  static RobotState from_vec(const V& s) {
    return {detail::at(s, 0), detail::at(s, 1), detail::at(s, 2), detail::at(s, 3), detail::at(s, 4)};
  }
  Vec2 position() const { return {x, y}; }
};
struct Control {  // core.hpp:54-59
  double v_ref{0.0}, omega_ref{0.0};
};
struct ControlBounds {  // core.hpp:61-74
  Control lo{-0.5, -2.0};
  Control hi{2.0, 2.0};
  Control clamp(const Control& u) const {
    auto c = [](double v, double lo, double hi) { return v < lo ? lo : (hi < v ? hi : v); };
    return {c(u.v_ref, lo.v_ref, hi.v_ref), c(u.omega_ref, lo.omega_ref, hi.omega_ref)};
  }
};
using ControlSequence = std::vector<Control>;

struct TerrainWeights {  // core.hpp:97-112
  Vector w;
  static TerrainWeights uniform(int m) { return {Vector(m, 1.0 / m)}; }
  int size() const { return static_cast<int>(w.size()); }
};

struct MppiConfig {  // mppi.hpp:16-26
  int samples{1024};
  int horizon{30};
  double lambda{0.1};
  Vec2 sigma_sim{0.09, 0.25};
  ControlBounds bounds;
  std::uint64_t seed{0};
  int threads{0};
  gpmppi_mppi_config c() const {
    return {samples, horizon, lambda, sigma_sim(0), sigma_sim(1), {bounds.lo.v_ref, bounds.lo.omega_ref},
            {bounds.hi.v_ref, bounds.hi.omega_ref}, seed, threads};
  }
};
struct NominalParams {  // dynamics.hpp:12-18
  double tau_v{0.5}, tau_omega{0.35}, dt{0.05};
};
struct Edd5Params {  // dynamics.hpp:36-45
  double alpha_l{1.0}, alpha_r{1.0}, x_icr{0.0}, y_icr_l{0.0}, y_icr_r{0.0};
  static Edd5Params ideal(double w) { return {1.0, 1.0, 0.0, -0.5 * w, 0.5 * w}; }
};
struct KernelParams {  // gp.hpp:12-22
  double signal_var{1.0};
  Vec4 lengthscales{1.0, 1.0, 1.0, 1.0};
  double noise_var{1e-4};
  bool operator==(const KernelParams& o) const {
    for (int i = 0; i < 4; ++i)
      if (lengthscales(i) != o.lengthscales(i)) return false;
    return signal_var == o.signal_var && noise_var == o.noise_var;
  }
};

// GpModel (gp.hpp:30-98): device-resident exact GP.
class GpModel {
 public:
  GpModel() = default;
  GpModel(GpModel&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}
  GpModel& operator=(GpModel&& o) noexcept {
    std::swap(h_, o.h_);
    return *this;
  }
  GpModel(const GpModel&) = delete;
  ~GpModel() { gpmppi_model_free(h_); }

  // inputs n×4 and outputs n×m, flat row-major
  static GpModel fit(const std::vector<double>& inputs, const std::vector<double>& outputs, int64_t m,
                     const std::vector<KernelParams>& kernels, int device = 0) {
    if (inputs.size() % 4 != 0 || inputs.empty())
      throw std::invalid_argument("GpModel::fit: inputs must be n x 4 with n >= 1");
    const int64_t n = static_cast<int64_t>(inputs.size() / 4);
    if (m < 1 || static_cast<int64_t>(outputs.size()) != n * m)
      throw std::invalid_argument("GpModel::fit: outputs must be n x m with m >= 1");
    if (static_cast<int64_t>(kernels.size()) != m)
      throw std::invalid_argument("GpModel::fit: one KernelParams per output column required");
    std::vector<double> k;
    for (const auto& p : kernels) {
      k.push_back(p.signal_var);
      for (double l : p.lengthscales) k.push_back(l);
      k.push_back(p.noise_var);
    }
    GpModel g;
    detail::check(gpmppi_model_fit(inputs.data(), outputs.data(), n, m, k.data(), device, &g.h_));
    return g;
  }
  // gp.hpp:34-35: any matrix type with rows(), cols(), (i, j) (Eigen::MatrixXd, Matrix)
  template <class MX, class MY, class = std::enable_if_t<detail::is_matrix<MX>::value && detail::is_matrix<MY>::value>>
  static GpModel fit(const MX& inputs, const MY& outputs, const std::vector<KernelParams>& kernels, int device = 0) {
    const long n = static_cast<long>(inputs.rows()), m = static_cast<long>(outputs.cols());
    if (n < 1 || inputs.cols() != 4) throw std::invalid_argument("GpModel::fit: inputs must be n x 4 with n >= 1");
    if (m < 1 || static_cast<long>(outputs.rows()) != n)
      throw std::invalid_argument("GpModel::fit: outputs must be n x m with m >= 1");
    std::vector<double> X(static_cast<size_t>(n * 4)), Y(static_cast<size_t>(n * m));
    for (long i = 0; i < n; ++i) {
      for (long d = 0; d < 4; ++d) X[i * 4 + d] = static_cast<double>(inputs(i, d));
      for (long j = 0; j < m; ++j) Y[i * m + j] = static_cast<double>(outputs(i, j));
    }
    return fit(X, Y, m, kernels, device);
  }
  static GpModel load(const std::string& path, int device = 0) {
    GpModel g;
    detail::check(gpmppi_model_load(path.c_str(), device, &g.h_));
    return g;
  }
  void save(const std::string& path) const { detail::check(gpmppi_model_save(h_, path.c_str())); }
  int n_points() const { return gpmppi_model_n_points(h_); }
  int n_outputs() const { return gpmppi_model_n_outputs(h_); }
  int n_groups() const { return gpmppi_model_n_groups(h_); }
  double group_jitter(int g) const { return gpmppi_model_group_jitter(h_, g); }
  double log_marginal_likelihood(int o) const {
    if (o < 0 || o >= n_outputs()) throw std::out_of_range("log_marginal_likelihood: output out of range");
    return gpmppi_model_log_marginal_likelihood(h_, o);
  }

  struct Prediction {  // gp.hpp:37-40
    Vector mean, var;
  };
  struct BatchPrediction {  // gp.hpp:43-46: S × n_outputs
    Matrix mean, var;
  };
  struct Workspace {};  // gp.hpp:49-53: the device keeps its own scratch

  // flat S×4 row-major queries
  BatchPrediction predict_batch(const std::vector<double>& queries) const {
    if (!h_) throw std::logic_error("GpModel::predict_batch: model not fitted");
    if (queries.size() % 4 != 0) throw std::invalid_argument("GpModel::predict_batch: queries must be S x 4");
    const long S = static_cast<long>(queries.size() / 4), m = n_outputs();
    BatchPrediction p{Matrix(S, m), Matrix(S, m)};
    detail::check(gpmppi_model_predict_batch(h_, queries.data(), S, p.mean.data(), p.var.data()));
    return p;
  }
  // gp.hpp:47: any S×4 matrix type
  template <class MQ, class = std::enable_if_t<detail::is_matrix<MQ>::value>>
  BatchPrediction predict_batch(const MQ& queries) const {
    if (queries.cols() != 4) throw std::invalid_argument("GpModel::predict_batch: queries must be S x 4");
    return predict_batch(flatten(queries));
  }
  // gp.hpp:41: one 4-vector query
  template <class V4>  // any 4-vector with q(i) or q[i]
  Prediction predict(const V4& q) const {
    std::vector<double> f(4);
    for (int d = 0; d < 4; ++d) f[d] = detail::at(q, d);
    const BatchPrediction b = predict_batch(f);
    Prediction p{Vector(n_outputs()), Vector(n_outputs())};
    for (long j = 0; j < n_outputs(); ++j) {
      p.mean(j) = b.mean(0, j);
      p.var(j) = b.var(0, j);
    }
    return p;
  }
  // gp.hpp:55-57: mean / var written into caller-sized S × n_outputs blocks
  template <class MQ, class MO>
  void predict_batch_into(const MQ& queries, MO& mean, MO& var, Workspace& /*ws*/) const {
    const BatchPrediction b = predict_batch(queries);
    if (static_cast<long>(mean.rows()) != b.mean.rows() || static_cast<long>(mean.cols()) != b.mean.cols() ||
        static_cast<long>(var.rows()) != b.var.rows() || static_cast<long>(var.cols()) != b.var.cols())
      throw std::invalid_argument("GpModel::predict_batch_into: mean/var must be S x n_outputs");
    for (long i = 0; i < b.mean.rows(); ++i)
      for (long j = 0; j < b.mean.cols(); ++j) {
        mean(i, j) = b.mean(i, j);
        var(i, j) = b.var(i, j);
      }
  }
  const gpmppi_model* handle() const { return h_; }
  static GpModel adopt(gpmppi_model* h) {  // takes ownership of a C-ABI handle
    GpModel g;
    g.h_ = h;
    return g;
  }

 private:
  template <class MQ>
  static std::vector<double> flatten(const MQ& q) {
    std::vector<double> f(static_cast<size_t>(q.rows()) * 4);
    for (long i = 0; i < static_cast<long>(q.rows()); ++i)
      for (long d = 0; d < 4; ++d) f[i * 4 + d] = static_cast<double>(q(i, d));
    return f;
  }
  gpmppi_model* h_ = nullptr;
};

// Prediction models (mppi.hpp:30-39)
struct GpEnsemble {
  const GpModel* model{nullptr};
  int n_terrains{0};
};
struct Edd5Baseline {
  Edd5Params params;
  double track_width{0.4};
};
struct UnicycleBaseline {};
struct NominalDynamic {};  // extension: zero-residual dynamic unicycle (BASELINE config 1)
using PredictionModel = std::variant<GpEnsemble, Edd5Baseline, UnicycleBaseline, NominalDynamic>;

// Tasks (costs.hpp:13-56, mppi.hpp:42-52)
struct Track {
  bool is_circle{false};
  Vec2 center{0.0, 0.0};
  double radius{0.0};
  std::vector<Vec2> waypoints;
  bool closed{true};
  double half_width{0.5};
  static Track circle_track(const Vec2& c, double r, double hw) { return {true, c, r, {}, true, hw}; }
  static Track polyline_track(std::vector<Vec2> pts, double hw, bool closed) {
    return {false, {0.0, 0.0}, 0.0, std::move(pts), closed, hw};
  }
  // costs.hpp:21-22 with the caller's 2-vector type (e.g. Eigen::Vector2d)
  template <class P, class = std::enable_if_t<!std::is_same_v<P, Vec2>>>
  static Track polyline_track(const std::vector<P>& pts, double hw, bool closed) {
    std::vector<Vec2> v;
    for (const auto& p : pts) v.push_back(Vec2(detail::at(p, 0), detail::at(p, 1)));
    return polyline_track(std::move(v), hw, closed);
  }
};
struct CircleObstacle {
  Vec2 center{0.0, 0.0};
  double radius{0.0};
};
struct TrackingWeights {
  double variance{0.1}, deviation{1.0}, slip{0.3}, safety{1.0}, speed{0.2};
};
struct AvoidanceWeights {
  double variance{0.1}, obstacle{1.0}, stage{0.5}, terminal{1.0};
};
struct GoalSpec {
  Vec2 position{0.0, 0.0};
  double capture_radius{0.5};
};
struct TrackingTask {
  const Track* track{nullptr};
  double v_desired{0.0};
  TrackingWeights weights;
};
struct AvoidanceTask {
  const std::vector<CircleObstacle>* obstacles{nullptr};
  GoalSpec goal;
  AvoidanceWeights weights;
  double high_cost{1e4};
};
// path tracking + tightened obstacle chance constraints (BASELINE config 2)
struct CombinedTask {
  const Track* track{nullptr};
  double v_desired{0.0};
  TrackingWeights weights;
  const std::vector<CircleObstacle>* obstacles{nullptr};
  double obstacle_weight{1.0};
};

struct StepDiagnostics {  // mppi.hpp:81-89
  double best_cost{0.0}, mean_cost{0.0}, ess{0.0}, weight_entropy{0.0};
  int nonfinite_samples{0};
  bool tightening_infeasible{false};
  double plan_ms{0.0};
  double command_ms{0.0};
};

namespace detail {
inline gpmppi_prediction_model model_c(const PredictionModel& model) {
  gpmppi_prediction_model pm{};
  if (auto* g = std::get_if<GpEnsemble>(&model)) {
    pm.kind = GPMPPI_MODEL_GP_ENSEMBLE;
    pm.gp = g->model ? g->model->handle() : nullptr;
    pm.n_terrains = g->n_terrains;
  } else if (auto* e = std::get_if<Edd5Baseline>(&model)) {
    pm.kind = GPMPPI_MODEL_EDD5;
    pm.edd5 = {e->params.alpha_l, e->params.alpha_r, e->params.x_icr, e->params.y_icr_l, e->params.y_icr_r};
    pm.track_width = e->track_width;
  } else if (std::holds_alternative<UnicycleBaseline>(model)) {
    pm.kind = GPMPPI_MODEL_UNICYCLE;
  } else {
    pm.kind = GPMPPI_MODEL_NOMINAL;
  }
  return pm;
}
inline void fill_diag(StepDiagnostics* diag, const gpmppi_diag& d) {
  if (!diag) return;
  diag->best_cost = d.best_cost;
  diag->mean_cost = d.mean_cost;
  diag->ess = d.ess;
  diag->weight_entropy = d.weight_entropy;
  diag->nonfinite_samples = d.nonfinite_samples;
  diag->tightening_infeasible = d.tightening_infeasible != 0;
  diag->plan_ms = d.plan_ms;
  diag->command_ms = d.command_ms;
}
}  // namespace detail

// Planner (mppi.hpp:96-143)
class Planner {
 public:
  Planner(const MppiConfig& cfg, PredictionModel model, NominalParams nominal, double p_x,
          int device = 0)
      : cfg_(cfg) {
    const gpmppi_prediction_model pm = detail::model_c(model);
    const gpmppi_mppi_config c = cfg.c();
    const gpmppi_nominal nom{nominal.tau_v, nominal.tau_omega, nominal.dt};
    detail::check(gpmppi_planner_create(&c, &pm, &nom, p_x, device, &h_));
  }
  Planner(Planner&& o) noexcept : cfg_(o.cfg_), h_(std::exchange(o.h_, nullptr)) {}
  Planner& operator=(Planner&& o) noexcept {
    std::swap(h_, o.h_);
    cfg_ = o.cfg_;
    return *this;
  }
  Planner(const Planner&) = delete;
  ~Planner() { gpmppi_planner_free(h_); }

  Control plan_step(const RobotState& x0, const TrackingTask& task, StepDiagnostics* diag = nullptr) {
    if (task.track == nullptr) throw std::invalid_argument("plan_step: tracking task needs a track");
    gpmppi_task t = base_task(GPMPPI_TASK_TRACKING, task.track, task.v_desired, task.weights);
    return run(x0, t, diag);
  }
  Control plan_step(const RobotState& x0, const AvoidanceTask& task, StepDiagnostics* diag = nullptr) {
    if (task.obstacles == nullptr) throw std::invalid_argument("plan_step: avoidance task needs an obstacle list");
    gpmppi_task t{};
    t.kind = GPMPPI_TASK_AVOIDANCE;
    set_obstacles(t, *task.obstacles);
    t.goal[0] = task.goal.position(0);
    t.goal[1] = task.goal.position(1);
    t.goal[2] = task.goal.capture_radius;
    t.avoidance = {task.weights.variance, task.weights.obstacle, task.weights.stage, task.weights.terminal};
    t.high_cost = task.high_cost;
    return run(x0, t, diag);
  }
  Control plan_step(const RobotState& x0, const CombinedTask& task, StepDiagnostics* diag = nullptr) {
    if (task.track == nullptr) throw std::invalid_argument("plan_step: tracking task needs a track");
    if (task.obstacles == nullptr) throw std::invalid_argument("plan_step: avoidance task needs an obstacle list");
    gpmppi_task t = base_task(GPMPPI_TASK_COMBINED, task.track, task.v_desired, task.weights);
    set_obstacles(t, *task.obstacles);
    t.avoidance.obstacle = task.obstacle_weight;
    t.high_cost = 1e4;
    return run(x0, t, diag);
  }

  // mppi.cpp:208-218
  void set_terrain_weights(const TerrainWeights& w) {
    detail::check(gpmppi_planner_set_terrain_weights(h_, w.w.data(), static_cast<int>(w.w.size())));
  }
  void set_terrain_weights(const std::vector<double>& w) {
    detail::check(gpmppi_planner_set_terrain_weights(h_, w.data(), static_cast<int>(w.size())));
  }
  TerrainWeights terrain_weights() const {
    std::vector<double> w(64);
    w.resize(gpmppi_planner_terrain_weights(h_, w.data()));
    return {Vector(std::move(w))};
  }
  ControlSequence nominal_sequence() const {
    std::vector<double> s(2 * cfg_.horizon);
    detail::check(gpmppi_planner_nominal_sequence(h_, s.data()));
    ControlSequence out(cfg_.horizon);
    for (int k = 0; k < cfg_.horizon; ++k) out[k] = {s[2 * k], s[2 * k + 1]};
    return out;
  }
  std::vector<Matrix5d> horizon_covariances() const {
    std::vector<Matrix5d> c(cfg_.horizon);
    detail::check(gpmppi_planner_horizon_covariances(h_, c[0].data()));  // [T][5][5] row-major
    return c;
  }
  Vector lane_radii() const {  // size N once a tracking tick has run, else empty
    std::vector<double> r(cfg_.horizon);
    r.resize(gpmppi_planner_lane_radii(h_, r.data()));
    return Vector(std::move(r));
  }
  Matrix obstacle_margins() const {  // N × n_obstacles
    std::vector<double> m(static_cast<size_t>(cfg_.horizon) * GPMPPI_MAX_OBSTACLES);
    const int O = gpmppi_planner_obstacle_margins(h_, m.data());
    Matrix out(O > 0 ? cfg_.horizon : 0, O);
    for (long i = 0; i < out.size(); ++i) out.data()[i] = m[i];
    return out;
  }
  const MppiConfig& config() const { return cfg_; }
  std::uint64_t tick() const { return gpmppi_planner_tick(h_); }
  gpmppi_planner* handle() { return h_; }

 private:
  static gpmppi_task base_task(int kind, const Track* tr, double v_des, const TrackingWeights& w) {
    gpmppi_task t{};
    t.kind = kind;
    track_c_.is_circle = tr->is_circle;
    track_c_.cx = tr->center(0);
    track_c_.cy = tr->center(1);
    track_c_.radius = tr->radius;
    wp_.clear();
    for (const auto& p : tr->waypoints) {
      wp_.push_back(p(0));
      wp_.push_back(p(1));
    }
    track_c_.n_waypoints = static_cast<int>(tr->waypoints.size());
    track_c_.waypoints = wp_.data();
    track_c_.closed = tr->closed;
    track_c_.half_width = tr->half_width;
    t.track = &track_c_;
    t.v_desired = v_des;
    t.tracking = {w.variance, w.deviation, w.slip, w.safety, w.speed};
    return t;
  }
  static void set_obstacles(gpmppi_task& t, const std::vector<CircleObstacle>& obs) {
    obs_.clear();
    for (const auto& o : obs) {
      obs_.push_back(o.center(0));
      obs_.push_back(o.center(1));
      obs_.push_back(o.radius);
    }
    t.obstacles = obs_.data();
    t.n_obstacles = static_cast<int>(obs.size());
  }
  Control run(const RobotState& x0, const gpmppi_task& t, StepDiagnostics* diag) {
    const Vec5 s = x0.vec();
    double cmd[2];
    gpmppi_diag d{};
    detail::check(gpmppi_planner_plan_step(h_, s.data(), &t, cmd, &d));
    detail::fill_diag(diag, d);
    return {cmd[0], cmd[1]};
  }

  MppiConfig cfg_;
  gpmppi_planner* h_ = nullptr;
  static inline thread_local gpmppi_track track_c_{};
  static inline thread_local std::vector<double> wp_;
  static inline thread_local std::vector<double> obs_;
};

// ---- models file GPMPPIM1 (harness.hpp:41-53, harness.cpp:249-284) ----
struct TrainedModels {
  bool has_gp{false};
  GpModel gp;
  Edd5Params edd5{Edd5Params::ideal(0.37)};
  NominalParams nominal;
};
inline TrainedModels load_models(const std::string& path, int device = 0) {
  gpmppi_edd5 e{};
  gpmppi_nominal n{};
  gpmppi_model* h = nullptr;
  detail::check(gpmppi_models_load(path.c_str(), device, &e, &n, &h));
  TrainedModels m;
  m.has_gp = h != nullptr;
  m.gp = GpModel::adopt(h);
  m.edd5 = {e.alpha_l, e.alpha_r, e.x_icr, e.y_icr_l, e.y_icr_r};
  m.nominal = {n.tau_v, n.tau_omega, n.dt};
  return m;
}
inline void save_models(const std::string& path, const TrainedModels& m) {
  const gpmppi_edd5 e{m.edd5.alpha_l, m.edd5.alpha_r, m.edd5.x_icr, m.edd5.y_icr_l, m.edd5.y_icr_r};
  const gpmppi_nominal n{m.nominal.tau_v, m.nominal.tau_omega, m.nominal.dt};
  detail::check(gpmppi_models_save(path.c_str(), &e, &n, m.has_gp ? m.gp.handle() : nullptr));
}

// ---- free functions (mppi.hpp:60-79), computed on the device ----
struct GaussianCorrection {  // core.hpp:89-94 (diagonal covariance, as combine_terrains fills it)
  Vec2 mean{0.0, 0.0};
  Matrix2d cov{};
  double trace() const { return cov(0, 0) + cov(1, 1); }
};
struct RolloutResult {  // mppi.hpp:53-56
  std::vector<RobotState> states;
  std::vector<GaussianCorrection> corrections;
};
// S perturbation blocks of N×2 (mppi.hpp:70: std::vector<Eigen::MatrixX2d>)
using Perturbations = std::vector<Matrix>;

inline RolloutResult rollout(const RobotState& x0, const ControlSequence& seq, const PredictionModel& model,
                             const std::vector<double>& weights, const NominalParams& nominal,
                             int device = 0) {
  const gpmppi_prediction_model pm = detail::model_c(model);
  const gpmppi_nominal nom{nominal.tau_v, nominal.tau_omega, nominal.dt};
  const int T = static_cast<int>(seq.size());
  std::vector<double> sq(2 * seq.size()), st(5 * (seq.size() + 1)), corr(4 * seq.size());
  for (size_t k = 0; k < seq.size(); ++k) {
    sq[2 * k] = seq[k].v_ref;
    sq[2 * k + 1] = seq[k].omega_ref;
  }
  const Vec5 x = x0.vec();
  const int R = pm.kind == GPMPPI_MODEL_GP_ENSEMBLE ? static_cast<int>(weights.size()) : 0;
  detail::check(gpmppi_rollout(&pm, &nom, weights.data(), R, x.data(), sq.data(), T, device, st.data(),
                               corr.data()));
  RolloutResult r;
  for (int k = 0; k <= T; ++k) r.states.push_back({st[5 * k], st[5 * k + 1], st[5 * k + 2], st[5 * k + 3], st[5 * k + 4]});
  for (int k = 0; k < T; ++k) {
    GaussianCorrection c;
    c.mean = {corr[4 * k], corr[4 * k + 1]};
    c.cov(0, 0) = corr[4 * k + 2];
    c.cov(1, 1) = corr[4 * k + 3];
    r.corrections.push_back(c);
  }
  return r;
}
// mppi.hpp:62-64 (TerrainWeights overload)
inline RolloutResult rollout(const RobotState& x0, const ControlSequence& seq, const PredictionModel& model,
                             const TerrainWeights& weights, const NominalParams& nominal, int device = 0) {
  return rollout(x0, seq, model, weights.w.std(), nominal, device);
}

// mppi.hpp:66-69: S blocks of N×2 (row k = (v noise, omega noise) of step k)
inline Perturbations sample_perturbations(const MppiConfig& cfg, std::uint64_t tick, int device = 0) {
  const gpmppi_mppi_config c = cfg.c();
  std::vector<double> e(static_cast<size_t>(cfg.samples) * cfg.horizon * 2);
  detail::check(gpmppi_sample_perturbations(&c, tick, device, e.data()));
  Perturbations out(cfg.samples, Matrix(cfg.horizon, 2));
  for (int s = 0; s < cfg.samples; ++s)
    for (long i = 0; i < 2L * cfg.horizon; ++i) out[s].data()[i] = e[static_cast<size_t>(s) * cfg.horizon * 2 + i];
  return out;
}

inline std::vector<double> trajectory_weights(const std::vector<double>& costs, double lambda, int device = 0) {
  std::vector<double> w(costs.size());
  detail::check(gpmppi_trajectory_weights(costs.data(), static_cast<int64_t>(costs.size()), lambda, device, w.data()));
  return w;
}
// mppi.hpp:71-72 with the caller's vector type (Eigen::VectorXd, Vector): returns the same type
template <class V, class = std::enable_if_t<detail::has_call1<V>::value>>
V trajectory_weights(const V& costs, double lambda, int device = 0) {
  std::vector<double> c(static_cast<size_t>(detail::length(costs)));
  for (size_t i = 0; i < c.size(); ++i) c[i] = detail::at(costs, static_cast<long>(i));
  const std::vector<double> w = trajectory_weights(c, lambda, device);
  V out(static_cast<long>(w.size()));
  for (size_t i = 0; i < w.size(); ++i) out(static_cast<long>(i)) = w[i];
  return out;
}

// mppi.hpp:74-76: eps = S blocks of N×2 (any matrix type), weights any vector type
template <class M, class W>
ControlSequence update_controls(const ControlSequence& nominal, const std::vector<M>& eps, const W& weights,
                                const ControlBounds& bounds, int device = 0) {
  static_assert(detail::is_matrix<M>::value, "update_controls: eps blocks need rows(), cols() and (i, j)");
  if (static_cast<long>(eps.size()) != detail::length(weights))
    throw std::invalid_argument("update_controls: one weight per sample required");
  const int T = static_cast<int>(nominal.size());
  std::vector<double> nom(2 * nominal.size()), e(eps.size() * 2 * nominal.size()), w(eps.size()),
      out(2 * nominal.size());
  for (int k = 0; k < T; ++k) {
    nom[2 * k] = nominal[k].v_ref;
    nom[2 * k + 1] = nominal[k].omega_ref;
  }
  for (size_t s = 0; s < eps.size(); ++s) {
    w[s] = detail::at(weights, static_cast<long>(s));
    for (int k = 0; k < T; ++k) {
      e[(s * T + k) * 2] = static_cast<double>(eps[s](k, 0));
      e[(s * T + k) * 2 + 1] = static_cast<double>(eps[s](k, 1));
    }
  }
  const double lo[2] = {bounds.lo.v_ref, bounds.lo.omega_ref}, hi[2] = {bounds.hi.v_ref, bounds.hi.omega_ref};
  detail::check(gpmppi_update_controls(nom.data(), T, e.data(), w.data(), static_cast<int64_t>(w.size()), lo, hi,
                                       device, out.data()));
  ControlSequence r(T);
  for (int k = 0; k < T; ++k) r[k] = {out[2 * k], out[2 * k + 1]};
  return r;
}

inline ControlSequence shift_horizon(const ControlSequence& seq, int device = 0) {
  if (seq.empty()) throw std::invalid_argument("shift_horizon: empty sequence");
  const int T = static_cast<int>(seq.size());
  std::vector<double> s(2 * seq.size()), out(2 * seq.size());
  for (int k = 0; k < T; ++k) {
    s[2 * k] = seq[k].v_ref;
    s[2 * k + 1] = seq[k].omega_ref;
  }
  detail::check(gpmppi_shift_horizon(s.data(), T, device, out.data()));
  ControlSequence r(T);
  for (int k = 0; k < T; ++k) r[k] = {out[2 * k], out[2 * k + 1]};
  return r;
}

// ---- scalar helpers (dynamics.hpp, uncertainty.hpp, core.hpp), host C++ in the library ----
inline double wrap_angle(double a) { return gpmppi_wrap_angle(a); }
inline RobotState step_nominal(const RobotState& s, const Control& u, const NominalParams& p) {
  const Vec5 x = s.vec();
  const double c[2] = {u.v_ref, u.omega_ref};
  const gpmppi_nominal n{p.tau_v, p.tau_omega, p.dt};
  Vec5 o;
  detail::check(gpmppi_step_nominal(x.data(), c, &n, o.data()));
  return RobotState::from_vec(o);
}
inline Matrix5d jacobian_nominal(const RobotState& s, const Control& u, const NominalParams& p) {
  const Vec5 x = s.vec();
  const double c[2] = {u.v_ref, u.omega_ref};
  const gpmppi_nominal n{p.tau_v, p.tau_omega, p.dt};
  Matrix5d J;
  detail::check(gpmppi_jacobian_nominal(x.data(), c, &n, J.data()));
  return J;
}
inline double chi2_quantile_2dof(double p) {
  double o = 0.0;
  detail::check(gpmppi_chi2_quantile_2dof(p, &o));
  return o;
}
inline double normal_quantile(double p) {
  double o = 0.0;
  detail::check(gpmppi_normal_quantile(p, &o));
  return o;
}
inline double normal_cdf(double x) { return gpmppi_normal_cdf(x); }

// B independent planners sharing one model (BASELINE config 4): robot b behaves as a
// Planner with seed seeds[b] (default cfg.seed + b). Combined tasks per robot.
class BatchPlanner {
 public:
  BatchPlanner(const MppiConfig& cfg, PredictionModel model, NominalParams nominal, double p_x, int robots,
               const std::vector<std::uint64_t>& seeds = {}, int device = 0)
      : cfg_(cfg), robots_(robots) {
    const gpmppi_prediction_model pm = detail::model_c(model);
    const gpmppi_mppi_config c = cfg.c();
    const gpmppi_nominal nom{nominal.tau_v, nominal.tau_omega, nominal.dt};
    if (!seeds.empty() && static_cast<int>(seeds.size()) != robots)
      throw std::invalid_argument("BatchPlanner: one seed per robot");
    detail::check(gpmppi_planner_create_batch(&c, &pm, &nom, p_x, robots, seeds.empty() ? nullptr : seeds.data(),
                                              device, &h_));
  }
  BatchPlanner(BatchPlanner&& o) noexcept : cfg_(o.cfg_), robots_(o.robots_), h_(std::exchange(o.h_, nullptr)) {}
  BatchPlanner(const BatchPlanner&) = delete;
  ~BatchPlanner() { gpmppi_planner_free(h_); }

  // one tick of every robot: states[b], tasks[b] -> commands[b]
  std::vector<Control> plan_step(const std::vector<RobotState>& x0, const std::vector<CombinedTask>& tasks,
                                 std::vector<StepDiagnostics>* diags = nullptr) {
    if (static_cast<int>(x0.size()) != robots_ || static_cast<int>(tasks.size()) != robots_)
      throw std::invalid_argument("BatchPlanner: one state and one task per robot");
    std::vector<double> xs(5 * x0.size());
    for (size_t b = 0; b < x0.size(); ++b) {
      const Vec5 v = x0[b].vec();
      for (int i = 0; i < 5; ++i) xs[5 * b + i] = v[i];
    }
    std::vector<gpmppi_track> tr(robots_);
    std::vector<std::vector<double>> wp(robots_), ob(robots_);
    std::vector<gpmppi_task> t(robots_);
    for (int b = 0; b < robots_; ++b) {
      const CombinedTask& k = tasks[b];
      if (!k.track || !k.obstacles) throw std::invalid_argument("BatchPlanner: combined task needs track and obstacles");
      tr[b] = {};
      tr[b].is_circle = k.track->is_circle;
      tr[b].cx = k.track->center(0);
      tr[b].cy = k.track->center(1);
      tr[b].radius = k.track->radius;
      for (const auto& p : k.track->waypoints) {
        wp[b].push_back(p(0));
        wp[b].push_back(p(1));
      }
      tr[b].n_waypoints = static_cast<int>(k.track->waypoints.size());
      tr[b].waypoints = wp[b].data();
      tr[b].closed = k.track->closed;
      tr[b].half_width = k.track->half_width;
      for (const auto& o : *k.obstacles) {
        ob[b].push_back(o.center(0));
        ob[b].push_back(o.center(1));
        ob[b].push_back(o.radius);
      }
      t[b] = {};
      t[b].kind = GPMPPI_TASK_COMBINED;
      t[b].track = &tr[b];
      t[b].v_desired = k.v_desired;
      t[b].tracking = {k.weights.variance, k.weights.deviation, k.weights.slip, k.weights.safety, k.weights.speed};
      t[b].obstacles = ob[b].data();
      t[b].n_obstacles = static_cast<int>(k.obstacles->size());
      t[b].avoidance.obstacle = k.obstacle_weight;
      t[b].high_cost = 1e4;
    }
    std::vector<double> cmd(2 * robots_);
    std::vector<gpmppi_diag> d(robots_);
    detail::check(gpmppi_planner_plan_step_batch(h_, xs.data(), t.data(), cmd.data(), d.data()));
    std::vector<Control> out(robots_);
    for (int b = 0; b < robots_; ++b) out[b] = {cmd[2 * b], cmd[2 * b + 1]};
    if (diags) {
      diags->resize(robots_);
      for (int b = 0; b < robots_; ++b) detail::fill_diag(&(*diags)[b], d[b]);
    }
    return out;
  }
  void set_terrain_weights(int robot, const std::vector<double>& w) {
    detail::check(gpmppi_planner_set_robot_terrain_weights(h_, robot, w.data(), static_cast<int>(w.size())));
  }
  int robots() const { return robots_; }
  std::uint64_t tick() const { return gpmppi_planner_tick(h_); }
  gpmppi_planner* handle() { return h_; }

 private:
  MppiConfig cfg_;
  int robots_;
  gpmppi_planner* h_ = nullptr;
};

}  // namespace gpmppi
