"""The reference's Python module surface (bindings/module.cpp:40-219, package `gpmppi`).

Same names, argument names, defaults, return shapes and exceptions as the pybind11
module `_gpmppi`, backed by libgpmppi_b200.so: the scalar helpers call the library's
host C++ (csrc/hostapi.cpp, the arithmetic the kernels share), the GP predicts on the
device, the closed-loop entry points run the device planner. The repository-root package
`gpmppi` re-exports this module so `import gpmppi` finds it, as with the reference.

Not provided: `benchmark_csv` (module.cpp:209-219, the CSV benchmark suite -- SURVEY §2
marks the CSV bench suite out of scope for this path).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _capi as A
from . import config as _config
from . import gpmppi as _G
from . import harness as _H

__doc__ = "Chance-constrained GP-MPPI planner for skid-steer robots"


def _vec(a, n, who):
    v = np.ascontiguousarray(a, dtype=np.float64).reshape(-1)
    if v.shape[0] != n:
        raise TypeError(f"{who}: expected {n} values")
    return v


def _mat2(a, who):
    m = np.ascontiguousarray(a, dtype=np.float64)
    if m.shape != (2, 2):
        raise TypeError(f"{who}: expected a 2x2 matrix")
    return m


# ---------------------------------------------------------------- core (module.cpp:40-50)
def wrap_angle(angle: float) -> float:
    return A.lib().gpmppi_wrap_angle(float(angle))


def body_frame_displacement(from_xy, from_theta: float, to_xy):
    f = np.array([*_vec(from_xy, 2, "body_frame_displacement"), float(from_theta), 0.0, 0.0])
    t = np.array([*_vec(to_xy, 2, "body_frame_displacement"), 0.0, 0.0, 0.0])
    out = np.empty(2)
    A.check(A.lib().gpmppi_body_frame_displacement(A.dptr(f), A.dptr(t), A.dptr(out)))
    return out


# ---------------------------------------------------------------- dynamics (module.cpp:52-85)
class NominalParams(_G.NominalParams):
    """dynamics.hpp:12-18; the keyword constructor validates (module.cpp:56-61)."""

    def __init__(self, tau_v: float = 0.5, tau_omega: float = 0.35, dt: float = 0.05):
        super().__init__(float(tau_v), float(tau_omega), float(dt))
        if not (self.tau_v > 0.0) or not (self.tau_omega > 0.0):
            raise ValueError("NominalParams: time constants must be positive")
        if not (self.dt > 0.0) or self.dt >= min(self.tau_v, self.tau_omega):
            raise ValueError("NominalParams: require 0 < dt < min(tau_v, tau_omega)")


def _nom_c(p):
    return A.NominalC(p.tau_v, p.tau_omega, p.dt)


def step_nominal(state, control, params):
    s, u, out = _vec(state, 5, "step_nominal"), _vec(control, 2, "step_nominal"), np.empty(5)
    pc = _nom_c(params)
    A.check(A.lib().gpmppi_step_nominal(A.dptr(s), A.dptr(u), C.byref(pc), A.dptr(out)))
    return out


def step_kinematic_unicycle(state, control, dt: float):
    s, u, out = _vec(state, 5, "step_kinematic_unicycle"), _vec(control, 2, "step_kinematic_unicycle"), np.empty(5)
    A.check(A.lib().gpmppi_step_kinematic_unicycle(A.dptr(s), A.dptr(u), float(dt), A.dptr(out)))
    return out


def jacobian_nominal(state, control, params):
    s, u, J = _vec(state, 5, "jacobian_nominal"), _vec(control, 2, "jacobian_nominal"), np.empty(25)
    pc = _nom_c(params)
    A.check(A.lib().gpmppi_jacobian_nominal(A.dptr(s), A.dptr(u), C.byref(pc), A.dptr(J)))
    return J.reshape(5, 5)


# ---------------------------------------------------------------- gp (module.cpp:86-140)
class KernelParams(_G.KernelParams):
    """gp.hpp:12-22; KernelParams(signal_var, lengthscales, noise_var) validates."""

    def __init__(self, signal_var: float = 1.0, lengthscales=(1.0, 1.0, 1.0, 1.0), noise_var: float = 1e-4):
        ls = tuple(float(v) for v in _vec(lengthscales, 4, "KernelParams"))
        super().__init__(float(signal_var), ls, float(noise_var))
        if not (self.signal_var > 0.0) or not (self.noise_var > 0.0) or not all(v > 0.0 for v in ls):
            raise ValueError("KernelParams: all parameters must be strictly positive")


class GpModel:
    """gp.hpp:30-98 over the device model handle (fit on the host in FP64 below n = 1024,
    on the device above; predictions on the device)."""

    def __init__(self, model: _G.GpModel):
        self._m = model

    @staticmethod
    def fit(inputs, outputs, kernels) -> "GpModel":
        X = np.ascontiguousarray(inputs, dtype=np.float64)
        Y = np.ascontiguousarray(outputs, dtype=np.float64)
        if X.ndim != 2 or X.shape[1] != 4:
            raise ValueError("GpModel::fit: inputs must be n x 4 with n >= 1")
        if Y.ndim != 2 or Y.shape[0] != X.shape[0]:
            raise ValueError("GpModel::fit: outputs must be n x m with m >= 1")
        if len(kernels) != Y.shape[1]:
            raise ValueError("GpModel::fit: one KernelParams per output required")
        return GpModel(_G.GpModel.fit(X, Y, [k.as_row() for k in kernels]))

    def predict(self, q):
        m, v = self._m.predict_batch(_vec(q, 4, "GpModel::predict").reshape(1, 4))
        return m[0].copy(), v[0].copy()

    def predict_batch(self, queries):
        Q = np.ascontiguousarray(queries, dtype=np.float64)
        if Q.ndim != 2 or Q.shape[1] != 4:
            raise ValueError("GpModel::predict_batch: queries must be S x 4")
        return self._m.predict_batch(Q)

    @property
    def n_points(self) -> int:
        return self._m.n_points

    @property
    def n_outputs(self) -> int:
        return self._m.n_outputs

    def log_marginal_likelihood(self, output: int) -> float:
        if not (0 <= output < self._m.n_outputs):
            raise IndexError("log_marginal_likelihood: output out of range")
        return self._m.log_marginal_likelihood(output)

    def save(self, path: str) -> None:
        self._m.save(path)

    @staticmethod
    def load(path: str) -> "GpModel":
        return GpModel(_G.GpModel.load(path))

    @property
    def device_model(self) -> _G.GpModel:
        """The planner-facing handle (for GpEnsemble)."""
        return self._m


def kernel_eval(a, b, params) -> float:
    av, bv = _vec(a, 4, "kernel_eval"), _vec(b, 4, "kernel_eval")
    k = np.array(params.as_row(), dtype=np.float64)
    out = C.c_double()
    A.check(A.lib().gpmppi_kernel_eval(A.dptr(av), A.dptr(bv), A.dptr(k), C.byref(out)))
    return out.value


def select_kernel_grid(inputs, outputs) -> KernelParams:
    """gp.cpp:274-366: shared-kernel LML grid (coarse 5x7x5 + refinement 5x7x5)."""
    k = _H.select_kernel_grid(inputs, outputs)
    return KernelParams(k.signal_var, k.lengthscales, k.noise_var)


def ensemble_combine(means, var_diags, weights):
    M = np.ascontiguousarray(means, dtype=np.float64)
    V = np.ascontiguousarray(var_diags, dtype=np.float64)
    w = np.ascontiguousarray(weights, dtype=np.float64).reshape(-1)
    if M.ndim != 2 or M.shape[1] != 2 or V.shape != M.shape:
        raise ValueError("ensemble_combine: size mismatch")
    mean, cov = np.empty(2), np.empty(4)
    A.check(A.lib().gpmppi_ensemble_combine(A.dptr(M), A.dptr(V), A.dptr(w), M.shape[0] if w.shape[0] == M.shape[0]
                                            else -1, A.dptr(mean), A.dptr(cov)))
    return mean, cov.reshape(2, 2)


# ---------------------------------------------------------------- terrain (module.cpp:142-159)
def project_simplex(z):
    v = np.ascontiguousarray(z, dtype=np.float64).reshape(-1)
    out = np.empty_like(v)
    A.check(A.lib().gpmppi_project_simplex(A.dptr(v), v.shape[0], A.dptr(out)))
    return out


def solve_terrain_weights(f_v, f_omega, y_v, y_omega, prev, gamma: float = 0.1):
    """module.cpp:143-159: a history buffer of the given rows, one weight solve."""
    fv, fw = np.atleast_2d(np.asarray(f_v, dtype=np.float64)), np.atleast_2d(np.asarray(f_omega, dtype=np.float64))
    rows, m = fv.shape
    buf = _H.HistoryBuffer(max(rows, 1), m)
    yv, yw = np.asarray(y_v, dtype=np.float64).reshape(-1), np.asarray(y_omega, dtype=np.float64).reshape(-1)
    for r in range(rows):
        buf.push((yv[r], yw[r]), np.column_stack([fv[r], fw[r]]))
    res = _H.solve_weights(buf, np.asarray(prev, dtype=np.float64),
                           _H.WeightSolverConfig(gamma=float(gamma)))
    return res.weights, res.objective


# ---------------------------------------------------------------- uncertainty (module.cpp:161-181)
def chi2_quantile_2dof(p: float) -> float:
    out = C.c_double()
    A.check(A.lib().gpmppi_chi2_quantile_2dof(float(p), C.byref(out)))
    return out.value


def normal_quantile(p: float) -> float:
    out = C.c_double()
    A.check(A.lib().gpmppi_normal_quantile(float(p), C.byref(out)))
    return out.value


def normal_cdf(x: float) -> float:
    return A.lib().gpmppi_normal_cdf(float(x))


def tighten_lane_radius(r: float, cov_xy, p_x: float = 0.95) -> float:
    c = _mat2(cov_xy, "tighten_lane_radius")
    out = C.c_double()
    A.check(A.lib().gpmppi_tighten_lane_radius(float(r), A.dptr(c), float(p_x), C.byref(out)))
    return out.value


def tighten_obstacle_distance(robot_xy, center, radius: float, cov_xy, p_x: float = 0.95):
    rx, cc = _vec(robot_xy, 2, "tighten_obstacle_distance"), _vec(center, 2, "tighten_obstacle_distance")
    c = _mat2(cov_xy, "tighten_obstacle_distance")
    d_bar, n, deg = C.c_double(), np.empty(2), C.c_int()
    A.check(A.lib().gpmppi_tighten_obstacle_distance(A.dptr(rx), A.dptr(cc), float(radius), A.dptr(c), float(p_x),
                                                      C.byref(d_bar), A.dptr(n), C.byref(deg), None))
    return d_bar.value, n, bool(deg.value)


# ---------------------------------------------------------------- harness (module.cpp:182-208)
def default_config_json() -> str:
    return _config.default_config_json()


def run_tracking(config_path: str = "", seed: int = 0, planner: str = "") -> dict:
    return _H.run_tracking(config_path, seed, planner)


def run_avoidance(config_path: str = "", seed: int = 0, planner: str = "") -> dict:
    return _H.run_avoidance(config_path, seed, planner)


__all__ = ["wrap_angle", "body_frame_displacement", "NominalParams", "step_nominal", "step_kinematic_unicycle",
           "jacobian_nominal", "KernelParams", "GpModel", "kernel_eval", "select_kernel_grid", "ensemble_combine",
           "project_simplex", "solve_terrain_weights", "chi2_quantile_2dof", "normal_quantile", "normal_cdf",
           "tighten_lane_radius", "tighten_obstacle_distance", "default_config_json", "run_tracking",
           "run_avoidance"]
