// Caller code written the way the reference's callers are (harness.cpp:190-244,
// mppi.cpp:115-160, module.cpp:98-121) -- Eigen-typed arguments -- compiled against
// include/gpmppi/planner.hpp with a minimal stand-in for the Eigen types it passes
// (rows(), cols(), v(i), m(i, j), resize), since Eigen itself is not in this image.
// Host-only calls run everywhere; the device calls need a GPU (exit 2 without one).
#include <cmath>
#include <cstdio>
#include <exception>
#include <type_traits>
#include <vector>

namespace Eigen {  // just enough of Eigen's dense interface for the calls below
using Index = long;
template <int R, int C>
class Matrix {
 public:
  Matrix() : r_(R > 0 ? R : 0), c_(C > 0 ? C : 0), d_((size_t)r_ * c_, 0.0) {}
  Matrix(Index r, Index c) : r_(r), c_(c), d_((size_t)(r * c), 0.0) {}
  explicit Matrix(Index n) : r_(C == 1 ? n : 1), c_(C == 1 ? 1 : n), d_((size_t)n, 0.0) {}
  template <int RR = R, int CC = C, class = std::enable_if_t<RR == 2 && CC == 1>>
  Matrix(double a, double b) : r_(2), c_(1), d_{a, b} {}
  template <int RR = R, int CC = C, class = std::enable_if_t<RR == 4 && CC == 1>>
  Matrix(double a, double b, double c, double d) : r_(4), c_(1), d_{a, b, c, d} {}
  double& operator()(Index i, Index j) { return d_[(size_t)(j * r_ + i)]; }  // column-major, as Eigen
  double operator()(Index i, Index j) const { return d_[(size_t)(j * r_ + i)]; }
  double& operator()(Index i) { return d_[(size_t)i]; }
  double operator()(Index i) const { return d_[(size_t)i]; }
  Index rows() const { return r_; }
  Index cols() const { return c_; }
  Index size() const { return r_ * c_; }
  void resize(Index r, Index c) {
    r_ = r;
    c_ = c;
    d_.assign((size_t)(r * c), 0.0);
  }

 private:
  Index r_, c_;
  std::vector<double> d_;
};
using MatrixXd = Matrix<-1, -1>;
using MatrixX2d = Matrix<-1, 2>;
using VectorXd = Matrix<-1, 1>;
using Vector2d = Matrix<2, 1>;
using Vector4d = Matrix<4, 1>;
}  // namespace Eigen

#include "gpmppi/planner.hpp"

using namespace gpmppi;

int main() {
  // ---- host-only (no device): value types, accessors, scalar helpers
  MppiConfig cfg;
  cfg.samples = 256;
  cfg.horizon = 12;
  cfg.seed = 5;
  const double sv = std::sqrt(cfg.sigma_sim(0)), sw = std::sqrt(cfg.sigma_sim(1));  // mppi.cpp:115
  const Track circle = Track::circle_track(Eigen::Vector2d(0.0, 0.0), 2.0, 0.4);   // costs.hpp:21
  const Track lane = Track::polyline_track(std::vector<Eigen::Vector2d>{Eigen::Vector2d(0.0, 0.0),
                                                                         Eigen::Vector2d(60.0, 0.0)},
                                           0.4, false);
  Eigen::Matrix<5, 1> sv5(5);
  sv5(0) = 2.0;
  sv5(2) = 1.5707963267948966;
  const RobotState x0 = RobotState::from_vec(sv5);
  KernelParams shared;
  shared.signal_var = 4e-3;
  shared.lengthscales = Eigen::Vector4d(0.8, 1.2, 0.8, 1.2);
  shared.noise_var = 1e-4;
  const RobotState nx = step_nominal(x0, Control{2.0, 0.0}, NominalParams{});
  const Matrix5d J = jacobian_nominal(x0, Control{1.0, 0.1}, NominalParams{});
  std::printf("host sigma=(%.3f, %.3f) circle=%d lane_wp=%zu x0=(%.1f, %.4f) ls2=%.1f nx_v=%.3f J33=%.2f q=%.6f\n",
              sv, sw, (int)circle.is_circle, lane.waypoints.size(), x0.x, x0.theta, shared.lengthscales(2), nx.v,
              J(3, 3), normal_quantile(0.975));
  try {
    // ---- harness.cpp:230-244: Eigen inputs n×4, outputs n×2M, one shared kernel
    const int n = 60, m = 3;
    Eigen::MatrixXd inputs(n, 4), outputs(n, 2 * m);
    for (int r = 0; r < n; ++r) {
      const double t = 0.37 * r;
      inputs(r, 0) = -0.5 + 2.5 * std::fmod(t, 1.0);
      inputs(r, 1) = -2.0 + 4.0 * std::fmod(1.7 * t, 1.0);
      inputs(r, 2) = -0.5 + 2.5 * std::fmod(2.3 * t, 1.0);
      inputs(r, 3) = -2.0 + 4.0 * std::fmod(3.1 * t, 1.0);
      for (int i = 0; i < m; ++i) {
        outputs(r, 2 * i) = 0.02 * std::sin(inputs(r, 0) + i) + 0.01 * inputs(r, 2);
        outputs(r, 2 * i + 1) = -0.015 * inputs(r, 3) + 0.005 * i;
      }
    }
    GpModel gp = GpModel::fit(inputs, outputs, std::vector<KernelParams>(2 * m, shared));
    // gp.hpp:41-57
    const auto one = gp.predict(Eigen::Vector4d(0.5, 0.1, 0.7, -0.2));
    Eigen::MatrixXd queries(5, 4);
    for (int i = 0; i < 5; ++i)
      for (int d = 0; d < 4; ++d) queries(i, d) = inputs(i, d);
    const auto batch = gp.predict_batch(queries);
    GpModel::Workspace ws;
    Eigen::MatrixXd mean(5, 2 * m), var(5, 2 * m);
    gp.predict_batch_into(queries, mean, var, ws);
    // mppi.hpp:60-79 with Eigen containers
    const std::vector<Matrix> eps = sample_perturbations(cfg, 0);
    std::vector<Eigen::MatrixX2d> eps_e(eps.size(), Eigen::MatrixX2d(cfg.horizon, 2));
    for (size_t s = 0; s < eps.size(); ++s)
      for (int k = 0; k < cfg.horizon; ++k) {
        eps_e[s](k, 0) = eps[s](k, 0);
        eps_e[s](k, 1) = eps[s](k, 1);
      }
    Eigen::VectorXd costs(cfg.samples);
    for (int s = 0; s < cfg.samples; ++s) costs(s) = 0.01 * (s % 17);
    const Eigen::VectorXd w = trajectory_weights(costs, 0.1);
    const ControlSequence seq(cfg.horizon, Control{0.5, 0.0});
    const ControlSequence upd = update_controls(seq, eps_e, w, cfg.bounds);
    TerrainWeights tw;
    tw.w = Eigen::VectorXd(m);
    for (int i = 0; i < m; ++i) tw.w(i) = 1.0 / m;
    const RolloutResult ro = rollout(x0, seq, GpEnsemble{&gp, m}, tw, NominalParams{});
    Planner planner(cfg, GpEnsemble{&gp, m}, NominalParams{}, 0.95);
    planner.set_terrain_weights(tw);
    StepDiagnostics d;
    const Control u = planner.plan_step(x0, TrackingTask{&circle, 2.0, {}}, &d);
    const auto radii = planner.lane_radii();
    std::printf("device pred=%.9f/%.9f batch=%.9f into=%.9f w0=%.6f upd0=%.6f states=%zu u=(%.6f, %.6f) "
                "radii=%ld cov00=%.3e ess=%.1f\n",
                one.mean(0), one.var(0), batch.mean(1, 2), mean(1, 2), w(0), upd[0].v_ref, ro.states.size(), u.v_ref,
                u.omega_ref, radii.size(), planner.horizon_covariances()[3](0, 0), d.ess);
    if (std::fabs(batch.mean(1, 2) - mean(1, 2)) > 0.0 || std::fabs(batch.var(4, 5) - var(4, 5)) > 0.0) return 4;
  } catch (const std::runtime_error& e) {
    std::printf("runtime_error: %s\n", e.what());
    return 2;
  } catch (const std::exception& e) {
    std::printf("exception: %s\n", e.what());
    return 3;
  }
  return 0;
}
