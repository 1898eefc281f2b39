// Drop-in usage of the B200 planner through the reference-shaped C++ API
// (include/gpmppi/planner.hpp): fit a GP, build a Planner, run plan_step on the
// tracking, avoidance and combined tasks. Prints one line per call.
#include <cmath>
#include <cstdio>
#include <exception>
#include <vector>

#include "gpmppi/planner.hpp"

int main() {
  using namespace gpmppi;
  try {
    const int n = 64, R = 3;
    std::vector<double> X(n * 4), Y(n * 2 * R);
    for (int i = 0; i < n; ++i) {
      const double t = i * 0.37;
      X[i * 4 + 0] = -0.5 + 2.5 * std::fmod(t, 1.0);
      X[i * 4 + 1] = -2.0 + 4.0 * std::fmod(t * 1.7, 1.0);
      X[i * 4 + 2] = -0.5 + 2.5 * std::fmod(t * 2.3, 1.0);
      X[i * 4 + 3] = -2.0 + 4.0 * std::fmod(t * 3.1, 1.0);
      for (int r = 0; r < R; ++r) {
        Y[i * 2 * R + 2 * r] = 0.02 * std::sin(X[i * 4] + r) + 0.01 * X[i * 4 + 2];
        Y[i * 2 * R + 2 * r + 1] = -0.015 * X[i * 4 + 3] + 0.005 * r;
      }
    }
    const KernelParams k{4e-3, {0.8, 1.2, 0.8, 1.2}, 1e-4};
    GpModel gp = GpModel::fit(X, Y, 2 * R, std::vector<KernelParams>(2 * R, k));
    MppiConfig cfg;
    cfg.samples = 512;
    cfg.horizon = 20;
    cfg.seed = 11;
    Planner planner(cfg, GpEnsemble{&gp, R}, NominalParams{}, 0.95);
    const Track lane = Track::polyline_track({{0.0, 0.0}, {60.0, 0.0}}, 0.4, false);
    const std::vector<CircleObstacle> obs = {{{3.0, 0.2}, 0.3}, {{5.0, -0.4}, 0.4}};
    StepDiagnostics d;
    Control u = planner.plan_step(RobotState{}, TrackingTask{&lane, 2.0, {}}, &d);
    std::printf("tracking  u=(%.6f, %.6f) ess=%.2f\n", u.v_ref, u.omega_ref, d.ess);
    u = planner.plan_step(RobotState{}, AvoidanceTask{&obs, {{8.0, 0.0}, 0.5}, {}, 1e4}, &d);
    std::printf("avoidance u=(%.6f, %.6f) best=%.4f\n", u.v_ref, u.omega_ref, d.best_cost);
    u = planner.plan_step(RobotState{}, CombinedTask{&lane, 2.0, {}, &obs, 1.0}, &d);
    std::printf("combined  u=(%.6f, %.6f) tick=%llu radii=%zu\n", u.v_ref, u.omega_ref,
                (unsigned long long)planner.tick(), planner.lane_radii().size());
    // free functions (mppi.hpp:60-79)
    const std::vector<double> w = trajectory_weights({0.0, 0.1}, 0.1);
    const ControlSequence seq = planner.nominal_sequence();
    const RolloutResult r = rollout(RobotState{}, seq, GpEnsemble{&gp, R}, {1.0 / 3, 1.0 / 3, 1.0 / 3}, NominalParams{});
    const Perturbations eps = sample_perturbations(cfg, 0);
    const ControlSequence up = update_controls(seq, eps, std::vector<double>(eps.size(), 1.0 / eps.size()), ControlBounds{});
    const ControlSequence sh = shift_horizon(seq);
    std::printf("free      w0=%.12f states=%zu eps=%zux%ld upd=%zu shift=%zu\n", w[0], r.states.size(), eps.size(),
                eps[0].rows(), up.size(), sh.size());
    // batched planner (config 4 API)
    BatchPlanner batch(cfg, GpEnsemble{&gp, R}, NominalParams{}, 0.95, 3);
    std::vector<Control> us = batch.plan_step({RobotState{}, RobotState{0.0, 0.1}, RobotState{0.0, -0.1}},
                                              {CombinedTask{&lane, 2.0, {}, &obs, 1.0}, CombinedTask{&lane, 1.5, {}, &obs, 1.0},
                                               CombinedTask{&lane, 1.0, {}, &obs, 1.0}});
    std::printf("batch     robots=%d u0=(%.6f, %.6f)\n", batch.robots(), us[0].v_ref, us[0].omega_ref);
  } catch (const std::runtime_error& e) {
    std::printf("runtime_error: %s\n", e.what());
    return 2;
  } catch (const std::exception& e) {
    std::printf("exception: %s\n", e.what());
    return 3;
  }
  return 0;
}
