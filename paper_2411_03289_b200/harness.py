"""Closed-loop drivers and terrain estimator around the B200 planner.

These are the hot path's callers: each tick plans on the GPU (`Planner.plan_step`), applies
the first control to the true-terrain simulator, pushes the measured transition into the
terrain history and re-solves the terrain weights on the host. Everything here is host
logic of a few hundred FLOPs per tick; the device work stays in the planner.

Follows, function by function:
  RngStream / derive_seed / splitmix64   rng.hpp:11-68 (mt19937_64 + Box-Muller, written out)
  arc_advance / step_nominal             dynamics.cpp:39-66
  TerrainProfile / step_true_terrain     dynamics.hpp:23-34, dynamics.cpp:129-139
  default_terrains                       config.cpp:116-124
  generate_training_data                 dynamics.cpp:141-170
  select_kernel_grid                     gp.cpp:274-366 (cells scored on the device)
  train_models (GP part)                 harness.cpp:190-243
  HistoryBuffer                          terrain.cpp:10-70
  project_simplex                        terrain.cpp:72-92
  solve_weights                          terrain.cpp:96-232
  per_terrain_mean_prediction            terrain.cpp:234-257
  Scenario / make_scenario               harness.hpp:16-31, harness.cpp:146-188
  random_obstacle_field                  harness.cpp:120-144
  run_tracking_experiment                harness.cpp:298-350
  run_avoidance_experiment               harness.cpp:352-421
  compute_rmse / summarize_latency       harness.cpp:286-296, 25-34

Not restated: the EDD5 least-squares fit (`fit_edd5`, dynamics.cpp:172-210; the ideal
parameters are used), the JSON config loader and the CSV bench suite (out of scope).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import gpmppi as G

_M64 = (1 << 64) - 1


# ----------------------------------------------------------------- rng.hpp
def splitmix64(x: int) -> int:  # rng.hpp:11-16
    x = (x + 0x9E3779B97F4A7C15) & _M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _M64
    return x ^ (x >> 31)


def derive_seed(seed: int, a: int, b: int = 0) -> int:  # rng.hpp:19-24
    h = splitmix64((seed ^ 0x6A09E667F3BCC909) & _M64)
    h = splitmix64(h ^ ((a * 0x9E3779B97F4A7C15) & _M64))
    return splitmix64(h ^ ((b * 0xBF58476D1CE4E5B9) & _M64))


class RngStream:
    """std::mt19937_64 (output pinned by the C++ standard) with the reference's draws
    (rng.hpp:29-68): 53-bit uniforms, scaled-double uniform_int, basic Box-Muller."""

    _N, _MM = 312, 156

    def __init__(self, seed: int):
        mt = [seed & _M64]
        for i in range(1, self._N):
            p = mt[-1]
            mt.append((6364136223846793005 * (p ^ (p >> 62)) + i) & _M64)
        self._mt = mt
        self._i = self._N
        self._spare = None

    def _twist(self):
        mt, n, m = self._mt, self._N, self._MM
        for i in range(n):
            y = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % n] & 0x7FFFFFFF)
            v = mt[(i + m) % n] ^ (y >> 1)
            if y & 1:
                v ^= 0xB5026F5AA96619E9
            mt[i] = v
        self._i = 0

    def next_u64(self) -> int:
        if self._i >= self._N:
            self._twist()
        y = self._mt[self._i]
        self._i += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & _M64

    def uniform01(self) -> float:
        return float(self.next_u64() >> 11) * 2.0 ** -53

    def uniform(self, lo: float, hi: float) -> float:
        return lo + (hi - lo) * self.uniform01()

    def uniform_int(self, lo: int, hi: int) -> int:
        r = lo + int(self.uniform01() * float(hi - lo + 1))
        return hi if r > hi else r

    def gaussian_pair(self):
        u1 = 1.0 - self.uniform01()
        u2 = self.uniform01()
        r = math.sqrt(-2.0 * math.log(u1))
        a = 2.0 * math.pi * u2
        return r * math.cos(a), r * math.sin(a)

    def gaussian(self) -> float:
        if self._spare is not None:
            z, self._spare = self._spare, None
            return z
        z0, z1 = self.gaussian_pair()
        self._spare = z1
        return z0


# ----------------------------------------------------------------- dynamics
_ARC_OMEGA_EPS = 1e-6


def wrap_angle(a: float) -> float:  # core.hpp:18-27
    if not math.isfinite(a):
        raise ValueError("wrap_angle: non-finite angle")
    r = math.remainder(a, 2.0 * math.pi)
    return r + 2.0 * math.pi if r <= -math.pi else r


def arc_advance(x, y, theta, vx, vy, omega, dt):  # dynamics.cpp:39-57
    if abs(omega) >= _ARC_OMEGA_EPS:
        s = math.sin(theta + omega * dt) - math.sin(theta)
        c = math.cos(theta + omega * dt) - math.cos(theta)
        x += (vx * s + vy * c) / omega
        y += (-vx * c + vy * s) / omega
    else:
        c0, s0 = math.cos(theta), math.sin(theta)
        half = 0.5 * omega * dt * dt
        ix = dt * c0 - half * s0
        iy = dt * s0 + half * c0
        x += vx * ix - vy * iy
        y += vx * iy + vy * ix
    return x, y, wrap_angle(theta + omega * dt)


def _check_finite(s, u, who):
    if not (all(math.isfinite(v) for v in s) and all(math.isfinite(v) for v in u)):
        raise ValueError(f"{who}: non-finite state or control")


def step_nominal(s, u, p: G.NominalParams):  # dynamics.cpp:59-66
    _check_finite(s, u, "step_nominal")
    x, y, th = arc_advance(s[0], s[1], s[2], s[3], 0.0, s[4], p.dt)
    return (x, y, th, s[3] + (p.dt / p.tau_v) * (u[0] - s[3]),
            s[4] + (p.dt / p.tau_omega) * (u[1] - s[4]))


@dataclass
class TerrainProfile:  # dynamics.hpp:23-34
    name: str = ""
    gain_v: float = 1.0
    gain_omega: float = 1.0
    tau_v_true: float = 0.5
    tau_omega_true: float = 0.35
    curvature_slip_c: float = 0.0
    noise_std_v: float = 0.0
    noise_std_omega: float = 0.0

    def validate(self):
        if not (self.gain_v > 0 and self.gain_omega > 0 and self.tau_v_true > 0
                and self.tau_omega_true > 0 and self.curvature_slip_c >= 0
                and self.noise_std_v >= 0 and self.noise_std_omega >= 0):
            raise ValueError(f"TerrainProfile {self.name!r}: bad parameters")


def default_terrains() -> List[TerrainProfile]:  # config.cpp:116-124
    return [TerrainProfile("tile", 0.97, 0.97, 0.45, 0.32, 0.05, 0.010, 0.020),
            TerrainProfile("asphalt", 0.92, 0.90, 0.55, 0.40, 0.15, 0.015, 0.030),
            TerrainProfile("grass", 0.82, 0.80, 0.70, 0.50, 0.35, 0.020, 0.040)]


def step_true_terrain(s, u, t: TerrainProfile, rng: RngStream, dt: float):  # dynamics.cpp:129-139
    _check_finite(s, u, "step_true_terrain")
    x, y, th = arc_advance(s[0], s[1], s[2], s[3], 0.0, s[4], dt)
    nv, nw = rng.gaussian_pair()
    omega_target = t.gain_omega * u[1] / (1.0 + t.curvature_slip_c * abs(s[3]))
    return (x, y, th,
            s[3] + (dt / t.tau_v_true) * (t.gain_v * u[0] - s[3]) + t.noise_std_v * nv,
            s[4] + (dt / t.tau_omega_true) * (omega_target - s[4]) + t.noise_std_omega * nw)


def generate_training_data(profile: TerrainProfile, nominal: G.NominalParams,
                           bounds: G.ControlBounds, n_points: int, rng: RngStream,
                           hold_min: int = 5, hold_max: int = 20):  # dynamics.cpp:141-170
    if n_points < 1:
        raise ValueError("generate_training_data: n_points must be >= 1")
    profile.validate()
    inputs = np.empty((n_points, 4))
    residuals = np.empty((n_points, 2))
    s = (0.0, 0.0, 0.0, 0.0, 0.0)
    u = (0.0, 0.0)
    hold = 0
    for i in range(n_points):
        if hold == 0:
            u = (rng.uniform(bounds.lo[0], bounds.hi[0]), rng.uniform(bounds.lo[1], bounds.hi[1]))
            hold = rng.uniform_int(hold_min, hold_max)
        hold -= 1
        inputs[i] = (s[3], s[4], u[0], u[1])
        nom = step_nominal(s, u, nominal)
        truth = step_true_terrain(s, u, profile, rng, nominal.dt)
        residuals[i] = (truth[3] - nom[3], truth[4] - nom[4])
        s = truth
    return inputs, residuals


# ----------------------------------------------------------------- GP hyperparameters
def select_kernel_grid(inputs, outputs, device: int = 0) -> G.KernelParams:
    """Shared-kernel LML grid search, coarse 5x7x5 then a 5x7x5 refinement (gp.cpp:274-366):
    every cell's Cholesky and LML on the device (gpmppi_select_kernel_grid, csrc/fit.cu)."""
    X = np.ascontiguousarray(inputs, dtype=np.float64)
    Y = np.ascontiguousarray(outputs, dtype=np.float64)
    if X.ndim != 2 or X.shape[1] != 4 or Y.ndim != 2 or Y.shape[0] != X.shape[0]:
        raise ValueError("select_kernel_grid: inputs n x 4 and outputs n x m required")
    k = np.empty(6)
    from . import _capi as A
    A.check(A.lib().gpmppi_select_kernel_grid(A.dptr(X), A.dptr(Y), X.shape[0], Y.shape[1], device,
                                              A.dptr(k), None))
    return G.KernelParams(float(k[0]), tuple(float(v) for v in k[1:5]), float(k[5]))


@dataclass
class ExperimentConfig:
    """The fields of config.hpp:85-110 the closed loop reads (JSON loading is out of scope)."""
    seed: int = 0
    planner: str = "gp"  # "gp" | "edd5" | "unicycle" (PlannerKind)
    nominal: G.NominalParams = field(default_factory=G.NominalParams)
    terrains: List[TerrainProfile] = field(default_factory=default_terrains)
    n_points: int = 300  # TrainingConfig
    hold_min: int = 5
    hold_max: int = 20
    grid_search: bool = True  # GpConfig
    fixed_kernel: G.KernelParams = field(default_factory=G.KernelParams)
    history: int = 20  # EstimatorConfig
    gamma: float = 0.1
    max_iters: int = 200
    tol: float = 1e-8
    p_x: float = 0.95
    tracking: G.TrackingWeights = field(default_factory=G.TrackingWeights)
    avoidance: G.AvoidanceWeights = field(default_factory=G.AvoidanceWeights)
    high_cost: float = 1e4
    mppi: G.MppiConfig = field(default_factory=G.MppiConfig)
    track_width: float = 0.37
    device: int = 0


def train_models(cfg: ExperimentConfig, seed: int) -> G.TrainedModels:
    """Per-terrain excitation data, a shared-input batch GP with 2M terrain-major outputs
    (harness.cpp:190-243), fitted on the device model handle. EDD5 stays at its ideal
    parameters (fit_edd5 is not restated)."""
    m, n = len(cfg.terrains), cfg.n_points
    per_terrain = []
    for i in range(m):
        rng = RngStream(derive_seed(seed, 100 + i))
        per_terrain.append(generate_training_data(cfg.terrains[i], cfg.nominal, cfg.mppi.bounds, n,
                                                  rng, cfg.hold_min, cfg.hold_max))
    inputs = np.stack([per_terrain[r % m][0][r] for r in range(n)])
    outputs = np.empty((n, 2 * m))
    for i in range(m):
        rng = RngStream(derive_seed(seed, 200 + i))
        for r in range(n):
            s = (0.0, 0.0, 0.0, inputs[r, 0], inputs[r, 1])
            u = (inputs[r, 2], inputs[r, 3])
            nom = step_nominal(s, u, cfg.nominal)
            truth = step_true_terrain(s, u, cfg.terrains[i], rng, cfg.nominal.dt)
            outputs[r, 2 * i] = truth[3] - nom[3]
            outputs[r, 2 * i + 1] = truth[4] - nom[4]
    kp = select_kernel_grid(inputs, outputs) if cfg.grid_search else cfg.fixed_kernel
    gp = G.GpModel.fit(inputs, outputs, [kp] * (2 * m), device=cfg.device)
    return G.TrainedModels(True, gp, G.Edd5Params.ideal(cfg.track_width), cfg.nominal)


# ----------------------------------------------------------------- terrain estimator
class HistoryBuffer:  # terrain.hpp:11-32, terrain.cpp:10-70
    def __init__(self, capacity: int, n_terrains: int):
        if capacity < 1 or n_terrains < 1:
            raise ValueError("HistoryBuffer: capacity and n_terrains must be >= 1")
        self._cap, self._m, self._head, self._size = capacity, n_terrains, 0, 0
        self._yv = np.zeros(capacity)
        self._yw = np.zeros(capacity)
        self._fv = np.zeros((capacity, n_terrains))
        self._fw = np.zeros((capacity, n_terrains))

    def push(self, measured, per_terrain):
        p = np.asarray(per_terrain, dtype=np.float64)
        if p.shape != (self._m, 2):
            raise ValueError("HistoryBuffer::push: expected one prediction row per terrain")
        h = self._head
        self._yv[h], self._yw[h] = measured[0], measured[1]
        self._fv[h], self._fw[h] = p[:, 0], p[:, 1]
        self._head = (h + 1) % self._cap
        self._size = min(self._size + 1, self._cap)

    def size(self) -> int:
        return self._size

    def capacity(self) -> int:
        return self._cap

    def n_terrains(self) -> int:
        return self._m

    def _order(self):  # oldest first
        start = (self._head - self._size + self._cap) % self._cap
        return (start + np.arange(self._size)) % self._cap

    def y_v(self):
        return self._yv[self._order()]

    def y_omega(self):
        return self._yw[self._order()]

    def f_v(self):
        return self._fv[self._order()]

    def f_omega(self):
        return self._fw[self._order()]


def project_simplex(z):  # terrain.cpp:72-92 (sorted-threshold rule)
    z = np.asarray(z, dtype=np.float64)
    if z.size < 1 or not np.isfinite(z).all():
        raise ValueError("project_simplex: need a finite non-empty vector")
    u = sorted(z.tolist(), reverse=True)
    cumsum, tau = 0.0, 0.0
    for i, ui in enumerate(u):
        cumsum += ui
        t = (cumsum - 1.0) / float(i + 1)
        if ui - t > 0.0:
            tau = t
    return np.maximum(z - tau, 0.0)


def on_simplex(w, tol: float) -> bool:  # core.hpp TerrainWeights::on_simplex
    w = np.asarray(w)
    return bool(w.size > 0 and np.isfinite(w).all() and w.min() >= -tol and abs(w.sum() - 1.0) <= tol)


@dataclass
class WeightSolverConfig:  # terrain.hpp:34-39
    gamma: float = 0.1
    max_iters: int = 200
    tol: float = 1e-8
    step0: float = 1.0


@dataclass
class WeightSolveResult:  # terrain.hpp:44-48
    weights: np.ndarray
    objective: float = 0.0
    buffer_empty: bool = False


class _Objective:  # terrain.cpp:96-120
    def __init__(self, buf: HistoryBuffer, prev, gamma):
        self.fv, self.fw = buf.f_v(), buf.f_omega()
        self.yv, self.yw = buf.y_v(), buf.y_omega()
        self.prev, self.gamma = np.asarray(prev, dtype=np.float64), gamma

    def __call__(self, w):
        rv, rw = self.yv - self.fv @ w, self.yw - self.fw @ w
        return float(rv @ rv + rw @ rw + self.gamma * np.abs(w - self.prev).sum())

    def subgradient(self, w):
        g = 2.0 * (self.fv.T @ (self.fv @ w - self.yv) + self.fw.T @ (self.fw @ w - self.yw))
        d = w - self.prev
        return g + self.gamma * np.sign(d)  # 0 on the kinks (minimising selection)


def _pairwise_line_min(obj: _Objective, w, i, j):  # terrain.cpp:122-157
    fvd, fwd = obj.fv[:, i] - obj.fv[:, j], obj.fw[:, i] - obj.fw[:, j]
    a2 = float(fvd @ fvd + fwd @ fwd)
    a1 = 2.0 * float(fvd @ (obj.fv @ w - obj.yv) + fwd @ (obj.fw @ w - obj.yw))
    t_lo, t_hi = -w[i], w[j]
    cand = [t_lo, t_hi]
    k1, k2 = obj.prev[i] - w[i], w[j] - obj.prev[j]
    if t_lo < k1 < t_hi:
        cand.append(k1)
    if t_lo < k2 < t_hi:
        cand.append(k2)
    if a2 > 0.0:
        for sgn in (-2.0, 0.0, 2.0):
            t = -(a1 + obj.gamma * sgn) / (2.0 * a2)
            if t_lo < t < t_hi:
                cand.append(t)
    best_t, best = 0.0, 0.0
    pi, pj, g = obj.prev[i], obj.prev[j], obj.gamma
    for t in cand:
        val = a2 * t * t + a1 * t + g * (abs(w[i] + t - pi) - abs(w[i] - pi)
                                         + abs(w[j] - t - pj) - abs(w[j] - pj))
        if val < best:
            best, best_t = val, t
    return best_t


def solve_weights(buf: HistoryBuffer, prev, cfg: WeightSolverConfig) -> WeightSolveResult:
    """min |Yv − Fv w|² + |Yω − Fω w|² + γ|w − prev|₁ over the simplex: projected
    subgradient with backtracking, then exact pairwise polishing (terrain.cpp:161-232)."""
    prev = np.asarray(prev, dtype=np.float64)
    if not on_simplex(prev, 1e-6):
        raise ValueError("solve_weights: prev weights must lie on the simplex")
    if cfg.gamma < 0.0 or not cfg.tol > 0.0:
        raise ValueError("solve_weights: gamma >= 0 and tol > 0 required")
    if buf.size() == 0:
        return WeightSolveResult(prev.copy(), 0.0, True)
    obj = _Objective(buf, prev, cfg.gamma)
    w = project_simplex(prev)
    fcur = obj(w)
    best_w, best = w, fcur
    grad_scale = max(float(np.abs(obj.subgradient(w)).max()), 1e-12)
    for t in range(cfg.max_iters):
        g = obj.subgradient(w)
        step = cfg.step0 / ((1.0 + t) * grad_scale)
        moved = False
        for _ in range(20):
            cand = project_simplex(w - step * g)
            fc = obj(cand)
            if fc <= fcur:
                w, fcur, moved = cand, fc, True
                break
            step *= 0.5
        if fcur < best:
            best, best_w = fcur, w
        if not moved:
            break
    m = buf.n_terrains()
    w, fcur = best_w.copy(), best
    for _ in range(100):
        improved = 0.0
        for i in range(m):
            for j in range(m):
                if i == j:
                    continue
                t = _pairwise_line_min(obj, w, i, j)
                if t == 0.0:
                    continue
                cand = w.copy()
                cand[i] = min(max(cand[i] + t, 0.0), 1.0)
                cand[j] = min(max(cand[j] - t, 0.0), 1.0)
                fc = obj(cand)
                if fc < fcur - 1e-16:
                    improved += fcur - fc
                    w, fcur = cand, fc
        if improved < 0.1 * cfg.tol:
            break
    if fcur < best:
        best, best_w = fcur, w
    out = project_simplex(best_w)
    return WeightSolveResult(out, obj(out), False)


def per_terrain_mean_prediction(model: G.GpModel, query, nominal: G.NominalParams):
    """Nominal next (v, ω) + each terrain's GP residual mean (terrain.cpp:234-257); the
    GP mean is evaluated by the device model."""
    m2 = model.n_outputs
    if m2 < 2 or m2 % 2:
        raise ValueError("per_terrain_mean_prediction: model must have 2M outputs")
    q = np.asarray(query, dtype=np.float64).reshape(4)
    v_next = q[0] + (nominal.dt / nominal.tau_v) * (q[2] - q[0])
    w_next = q[1] + (nominal.dt / nominal.tau_omega) * (q[3] - q[1])
    mean, _ = model.predict(q)
    mean = np.asarray(mean).reshape(m2)
    return np.column_stack([v_next + mean[0::2], w_next + mean[1::2]])


# ----------------------------------------------------------------- scenarios
def _point_segment_distance(p, a, b):  # costs.cpp:9-16
    ab = b - a
    len2 = float(ab @ ab)
    if len2 <= 0.0:
        return float(np.linalg.norm(p - a))
    t = min(max(float((p - a) @ ab) / len2, 0.0), 1.0)
    return float(np.linalg.norm(p - (a + t * ab)))


def centerline_distance(track: G.Track, xy) -> float:  # costs.cpp:62-74
    p = np.asarray(xy, dtype=np.float64)
    if track.is_circle:
        return abs(float(np.linalg.norm(p - np.asarray(track.center))) - track.radius)
    wp = track.waypoints
    n = len(wp)
    nseg = n if track.closed else n - 1
    return min(_point_segment_distance(p, wp[i], wp[(i + 1) % n]) for i in range(nseg))


@dataclass
class Scenario:  # harness.hpp:16-31
    kind: str = "tracking"
    track: G.Track = field(default_factory=lambda: G.Track.circle_track((0.0, 0.0), 2.0, 0.4))
    v_desired: float = 2.0
    start: tuple = (2.0, 0.0, math.pi / 2, 0.0, 0.0)
    goal: G.GoalSpec = field(default_factory=lambda: G.GoalSpec((8.0, 0.0), 0.5))
    obstacles: list = field(default_factory=list)
    schedule: list = field(default_factory=lambda: [(0.0, 0)])  # (time_s, terrain)
    distance_budget: float = 100.0
    max_duration: float = 120.0

    def terrain_at(self, t: float) -> int:  # harness.cpp:112-118
        cur = self.schedule[0][1]
        for ts, ter in self.schedule:
            if ts <= t:
                cur = ter
        return cur


def random_obstacle_field(rng: RngStream, count=5, x_range=(1.5, 6.5), y_range=(-2.5, 2.5),
                          radius_range=(0.25, 0.5), min_gap=0.5, start=(0.0, 0.0),
                          goal: G.GoalSpec = None):  # harness.cpp:120-144
    goal = goal or G.GoalSpec((8.0, 0.0), 0.5)
    if count < 0:
        raise ValueError("random_obstacle_field: count must be >= 0")
    if not (x_range[1] > x_range[0] and y_range[1] > y_range[0]
            and radius_range[1] >= radius_range[0] and radius_range[0] > 0.0):
        raise ValueError("random_obstacle_field: bad bounds or radii")
    out, attempts = [], 0
    while len(out) < count:
        attempts += 1
        if attempts > 10000:
            raise RuntimeError("random_obstacle_field: rejection sampling exceeded 10000 attempts")
        cx, cy = rng.uniform(*x_range), rng.uniform(*y_range)
        r = rng.uniform(*radius_range)
        if math.hypot(cx - start[0], cy - start[1]) < r + min_gap:
            continue
        if math.hypot(cx - goal.position[0], cy - goal.position[1]) < r + goal.capture_radius + min_gap:
            continue
        out.append(G.CircleObstacle((cx, cy), r))
    return out


def make_scenario(kind: str = "tracking", track: str = "circle", seed: int = 0,
                  v_desired: float = 2.0, schedule=None, distance_budget: float = 100.0,
                  max_duration: float = 120.0, n_obstacles: int = 5,
                  goal: G.GoalSpec = None, geometry: dict = None, start=None, obstacles=None,
                  random_obstacles: dict = None) -> Scenario:
    """Scenario from the config's geometry (config.hpp:43-54, harness.cpp:146-188).
    geometry / random_obstacles take the JSON config's sections (paper_2411_03289_b200.config);
    start (x, y, theta) overrides the canonical start; obstacles (list of (x, y, r)) replaces
    the random field."""
    goal = goal or G.GoalSpec((8.0, 0.0), 0.5)
    geo = geometry or {}
    circ = {"center": [0.0, 0.0], "radius": 2.0, "half_width": 0.4, **geo.get("circle", {})}
    sq = {"center": [0.0, 0.0], "side": 6.25, "half_width": 0.4, **geo.get("square", {})}
    lane = {"from": [0.0, 0.0], "to": [60.0, 0.0], "half_width": 0.4, **geo.get("lane", {})}
    sc = Scenario(kind=kind, v_desired=v_desired, goal=goal,
                  schedule=list(schedule or [(0.0, 0)]), distance_budget=distance_budget,
                  max_duration=max_duration)
    if track == "circle":
        c, r = circ["center"], circ["radius"]
        sc.track = G.Track.circle_track(tuple(c), r, circ["half_width"])
        st = (c[0] + r, c[1], 0.5 * math.pi)
    elif track == "square":
        h, c = 0.5 * sq["side"], sq["center"]
        sc.track = G.Track.polyline_track([(c[0] + h, c[1] - h), (c[0] + h, c[1] + h), (c[0] - h, c[1] + h),
                                           (c[0] - h, c[1] - h)], sq["half_width"], True)
        st = (c[0], c[1] - h, 0.0)
    elif track == "lane":
        a, b = lane["from"], lane["to"]
        sc.track = G.Track.polyline_track([tuple(a), tuple(b)], lane["half_width"], False)
        st = (a[0], a[1], math.atan2(b[1] - a[1], b[0] - a[0]))
    else:
        raise ValueError(f"make_scenario: unknown track {track!r}")
    if kind == "avoidance":
        st = (0.0, 0.0, math.atan2(goal.position[1], goal.position[0]))
    elif kind != "tracking":
        raise ValueError(f"make_scenario: unknown kind {kind!r}")
    if start is not None:
        st = tuple(start)
    sc.start = (st[0], st[1], wrap_angle(st[2]), 0.0, 0.0)
    if kind == "avoidance":
        if obstacles is not None:
            sc.obstacles = [G.CircleObstacle((float(o[0]), float(o[1])), float(o[2])) for o in obstacles]
        else:
            ro = {"count": n_obstacles, "x_min": 1.5, "x_max": 6.5, "y_min": -2.5, "y_max": 2.5,
                  "radius_min": 0.25, "radius_max": 0.5, "min_gap": 0.5, **(random_obstacles or {})}
            rng = RngStream(derive_seed(seed, 3))
            sc.obstacles = random_obstacle_field(rng, ro["count"], (ro["x_min"], ro["x_max"]),
                                                 (ro["y_min"], ro["y_max"]), (ro["radius_min"], ro["radius_max"]),
                                                 ro["min_gap"], start=sc.start[:2], goal=goal)
    return sc


# ----------------------------------------------------------------- closed loops
@dataclass
class LatencyStats:  # harness.hpp:53-57
    mean_ms: float = 0.0
    median_ms: float = 0.0
    max_ms: float = 0.0


@dataclass
class RunMetrics:  # harness.hpp:59-71
    rmse: float = 0.0
    success: bool = False
    time_to_goal: float = 0.0
    min_obstacle_clearance: float = math.inf
    mean_speed: float = 0.0
    collision_count: int = 0
    ticks: int = 0
    aborted: bool = False
    abort_reason: str = ""
    latency: LatencyStats = field(default_factory=LatencyStats)


@dataclass
class TraceRow:  # harness.hpp:74-81
    tick: int
    t: float
    state: tuple
    command: tuple
    best_cost: float
    mean_cost: float
    ess: float
    entropy: float
    terrain_weights: np.ndarray


def summarize_latency(ms) -> LatencyStats:  # harness.cpp:25-34
    if not ms:
        return LatencyStats()
    s = sorted(ms)
    mid = len(s) // 2
    med = s[mid] if len(s) % 2 else 0.5 * (s[mid - 1] + s[mid])
    return LatencyStats(sum(ms) / len(ms), med, max(ms))


def compute_rmse(path, track: G.Track) -> float:  # harness.cpp:286-296
    if len(path) == 0:
        raise ValueError("compute_rmse: empty path")
    return math.sqrt(sum(centerline_distance(track, p) ** 2 for p in path) / len(path))


def _make_planner(cfg: ExperimentConfig, models: G.TrainedModels, seed: int):  # harness.cpp:36-59
    m = len(cfg.terrains)
    if cfg.planner == "gp":
        if not models.has_gp:
            raise ValueError("gp planner requested but models carry no GP")
        pm = G.GpEnsemble(models.gp, m)
    elif cfg.planner == "edd5":
        pm = G.Edd5Baseline(models.edd5, cfg.track_width)
    elif cfg.planner == "unicycle":
        pm = G.UnicycleBaseline()
    else:
        raise ValueError(f"bad planner kind {cfg.planner!r}")
    mc = G.MppiConfig(**{**cfg.mppi.__dict__, "seed": derive_seed(seed, 2)})
    return G.Planner(mc, pm, cfg.nominal, cfg.p_x, device=cfg.device)


class _Loop:  # harness.cpp:61-110 (LoopState, apply_truth_step, update_terrain_estimate)
    def __init__(self, cfg, scenario, models, seed, trace):
        self.cfg, self.sc, self.models, self.trace = cfg, scenario, models, trace
        self.truth = tuple(scenario.start)
        self.rng = RngStream(derive_seed(seed, 1))
        self.t = 0.0
        self.path_len = 0.0
        self.positions = []
        self.latencies = []
        m = len(cfg.terrains)
        self.buf = HistoryBuffer(cfg.history, m)
        self.w = np.full(m, 1.0 / m)
        self.planner = _make_planner(cfg, models, seed)
        self.estimate = cfg.planner == "gp"
        if self.estimate:
            self.planner.set_terrain_weights(self.w)
        self.max_ticks = int(math.ceil(scenario.max_duration / cfg.nominal.dt)) + 1

    def plan(self, task, metrics):
        diag = G.StepDiagnostics()
        try:
            u = self.planner.plan_step(np.asarray(self.truth), task, diag)
        except Exception as e:  # harness.cpp:321-325 catches std::exception
            metrics.aborted, metrics.abort_reason = True, str(e)
            return None, diag
        self.latencies.append(diag.plan_ms)
        return (float(u[0]), float(u[1])), diag

    def truth_step(self, u):
        prev = self.truth
        ter = self.cfg.terrains[self.sc.terrain_at(self.t)]
        self.truth = step_true_terrain(prev, u, ter, self.rng, self.cfg.nominal.dt)
        self.t += self.cfg.nominal.dt
        self.path_len += math.hypot(self.truth[0] - prev[0], self.truth[1] - prev[1])
        self.positions.append((self.truth[0], self.truth[1]))
        return prev

    def update_estimate(self, prev, u):
        if not self.estimate:
            return
        q = (prev[3], prev[4], u[0], u[1])
        pred = per_terrain_mean_prediction(self.models.gp, q, self.models.nominal)
        self.buf.push((self.truth[3], self.truth[4]), pred)
        scfg = WeightSolverConfig(self.cfg.gamma, self.cfg.max_iters, self.cfg.tol, 1.0)
        self.w = solve_weights(self.buf, self.w, scfg).weights
        self.planner.set_terrain_weights(self.w)

    def push_trace(self, tick, u, diag):
        if self.trace is not None:
            self.trace.append(TraceRow(tick, self.t, self.truth, u, diag.best_cost, diag.mean_cost,
                                       diag.ess, diag.weight_entropy, self.w.copy()))


def run_tracking_experiment(cfg: ExperimentConfig, scenario: Scenario, models: G.TrainedModels,
                            seed: int, trace: Optional[list] = None) -> RunMetrics:
    """Closed-loop tracking until the distance budget (harness.cpp:298-350)."""
    if scenario.kind != "tracking":
        raise ValueError("run_tracking_experiment: scenario kind mismatch")
    lp = _Loop(cfg, scenario, models, seed, trace)
    task = G.TrackingTask(scenario.track, scenario.v_desired, cfg.tracking)
    met = RunMetrics()
    tick = 0
    while tick < lp.max_ticks and lp.path_len < scenario.distance_budget:
        u, diag = lp.plan(task, met)
        if u is None:
            break
        prev = lp.truth_step(u)
        met.ticks += 1
        if not all(math.isfinite(v) for v in lp.truth):
            met.aborted, met.abort_reason = True, "non-finite state"
            break
        if centerline_distance(scenario.track, lp.truth[:2]) > 25.0:
            met.aborted, met.abort_reason = True, "diverged from track"
            break
        lp.update_estimate(prev, u)
        lp.push_trace(tick, u, diag)
        tick += 1
    if lp.positions:
        met.rmse = compute_rmse(lp.positions, scenario.track)
    met.success = not met.aborted and lp.path_len >= scenario.distance_budget
    met.time_to_goal = lp.t if met.success else 0.0
    met.mean_speed = lp.path_len / lp.t if lp.t > 0.0 else 0.0
    met.latency = summarize_latency(lp.latencies)
    return met


def run_avoidance_experiment(cfg: ExperimentConfig, scenario: Scenario, models: G.TrainedModels,
                             seed: int, trace: Optional[list] = None) -> RunMetrics:
    """Closed-loop start-to-goal run; success = capture with zero physical collisions
    (harness.cpp:352-421)."""
    if scenario.kind != "avoidance":
        raise ValueError("run_avoidance_experiment: scenario kind mismatch")
    lp = _Loop(cfg, scenario, models, seed, trace)
    task = G.AvoidanceTask(scenario.obstacles, scenario.goal, cfg.avoidance, cfg.high_cost)
    met = RunMetrics()
    reached, in_prev = False, False
    for tick in range(lp.max_ticks):
        u, diag = lp.plan(task, met)
        if u is None:
            break
        margins = lp.planner.obstacle_margins()
        if np.size(margins) > 0 and float(np.min(margins)) < -1e-12:
            raise RuntimeError("tightening produced a negative margin")
        prev = lp.truth_step(u)
        met.ticks += 1
        if not all(math.isfinite(v) for v in lp.truth):
            met.aborted, met.abort_reason = True, "non-finite state"
            break
        clearance = min((math.hypot(lp.truth[0] - o.center[0], lp.truth[1] - o.center[1]) - o.radius
                         for o in scenario.obstacles), default=math.inf)
        met.min_obstacle_clearance = min(met.min_obstacle_clearance, clearance)
        hit = clearance < 0.0
        if hit and not in_prev:
            met.collision_count += 1
        in_prev = hit
        lp.update_estimate(prev, u)
        lp.push_trace(tick, u, diag)
        gx, gy = scenario.goal.position
        if math.hypot(lp.truth[0] - gx, lp.truth[1] - gy) <= scenario.goal.capture_radius:
            reached = True
            break
    met.success = reached and met.collision_count == 0 and not met.aborted
    met.time_to_goal = lp.t if reached else 0.0
    met.mean_speed = lp.path_len / lp.t if lp.t > 0.0 else 0.0
    met.latency = summarize_latency(lp.latencies)
    return met


# ----------------------------------------------------------------- Python entry points
def _metrics_to_dict(m: RunMetrics) -> dict:  # module.cpp:22-36
    return {"rmse": m.rmse, "success": m.success, "time_to_goal": m.time_to_goal,
            "min_obstacle_clearance": m.min_obstacle_clearance, "mean_speed": m.mean_speed,
            "collision_count": m.collision_count, "ticks": m.ticks, "aborted": m.aborted,
            "abort_reason": m.abort_reason, "latency_median_ms": m.latency.median_ms}


def _run(kind: str, config_path: str, seed: int, planner: str, **scenario):
    """module.cpp:183-208: the JSON config (or the default one), seed and planner overrides,
    models trained unless the planner is the unicycle, then one closed-loop run."""
    from . import config as CF
    jc = CF.load_config(config_path) if config_path else CF.default_config()
    jc["seed"] = seed
    if planner:
        CF.planner_kind(planner)
        jc["planner"] = planner
    jc["scenario"]["kind"] = kind
    cfg, sc_kwargs = CF.to_experiment(jc)
    sc_kwargs.update(scenario)
    models = G.TrainedModels() if cfg.planner == "unicycle" else train_models(cfg, seed)
    sc = make_scenario(seed=seed, **sc_kwargs)
    run = run_tracking_experiment if kind == "tracking" else run_avoidance_experiment
    return _metrics_to_dict(run(cfg, sc, models, seed))


def run_tracking(config_path: str = "", seed: int = 0, planner: str = "", **scenario) -> dict:
    """module.cpp:183-196: config, train, closed-loop tracking, metrics dict."""
    return _run("tracking", config_path, seed, planner, **scenario)


def run_avoidance(config_path: str = "", seed: int = 0, planner: str = "", **scenario) -> dict:
    """module.cpp:197-210: config, train, closed-loop avoidance, metrics dict."""
    return _run("avoidance", config_path, seed, planner, **scenario)
