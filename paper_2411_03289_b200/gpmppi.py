"""Host-side mirror of the reference planner API over the C ABI.

Same names, argument meaning and error behaviour as the reference's C++ API
(/root/reference/proj/include/gpmppi/{mppi,gp,costs,dynamics}.hpp) and its
pybind11 module (bindings/module.cpp): invalid arguments raise ValueError
(std::invalid_argument), factorisation / IO failures raise RuntimeError
(std::runtime_error). All compute runs on the GPU through libgpmppi_b200.so.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _capi as A


def _f64(a, shape=None):
    out = np.ascontiguousarray(a, dtype=np.float64)
    if shape is not None:
        out = out.reshape(shape)
    return out


# ----------------------------------------------------------------- value types
@dataclass
class KernelParams:  # gp.hpp:12-22
    signal_var: float = 1.0
    lengthscales: Sequence[float] = (1.0, 1.0, 1.0, 1.0)
    noise_var: float = 1e-4

    def as_row(self):
        return [self.signal_var, *list(self.lengthscales), self.noise_var]


@dataclass
class NominalParams:  # dynamics.hpp:12-18
    tau_v: float = 0.5
    tau_omega: float = 0.35
    dt: float = 0.05


@dataclass
class ControlBounds:  # core.hpp:61-74
    lo: tuple = (-0.5, -2.0)
    hi: tuple = (2.0, 2.0)


@dataclass
class MppiConfig:  # mppi.hpp:16-26
    samples: int = 1024
    horizon: int = 30
    lam: float = 0.1
    sigma_sim: tuple = (0.09, 0.25)
    bounds: ControlBounds = field(default_factory=ControlBounds)
    seed: int = 0
    threads: int = 0

    def to_c(self):
        return A.MppiConfigC(self.samples, self.horizon, self.lam, self.sigma_sim[0],
                             self.sigma_sim[1], (C.c_double * 2)(*self.bounds.lo),
                             (C.c_double * 2)(*self.bounds.hi), self.seed, self.threads)


@dataclass
class Edd5Params:  # dynamics.hpp:36-45
    alpha_l: float = 1.0
    alpha_r: float = 1.0
    x_icr: float = 0.0
    y_icr_l: float = 0.0
    y_icr_r: float = 0.0

    @staticmethod
    def ideal(track_width):
        return Edd5Params(1.0, 1.0, 0.0, -0.5 * track_width, 0.5 * track_width)


@dataclass
class TrackingWeights:  # costs.hpp:34-40
    variance: float = 0.1
    deviation: float = 1.0
    slip: float = 0.3
    safety: float = 1.0
    speed: float = 0.2


@dataclass
class AvoidanceWeights:  # costs.hpp:44-50
    variance: float = 0.1
    obstacle: float = 1.0
    stage: float = 0.5
    terminal: float = 1.0


@dataclass
class GoalSpec:  # costs.hpp:52-55
    position: tuple = (0.0, 0.0)
    capture_radius: float = 0.5


@dataclass
class CircleObstacle:  # costs.hpp:29-32
    center: tuple
    radius: float


class Track:  # costs.hpp:13-27
    def __init__(self, is_circle, center=(0.0, 0.0), radius=0.0, waypoints=None, closed=True,
                 half_width=0.5):
        self.is_circle = bool(is_circle)
        self.center = tuple(center)
        self.radius = float(radius)
        self.waypoints = None if waypoints is None else _f64(waypoints, (-1, 2))
        self.closed = bool(closed)
        self.half_width = float(half_width)

    @staticmethod
    def circle_track(center, radius, half_width):
        return Track(True, center=center, radius=radius, half_width=half_width)

    @staticmethod
    def polyline_track(points, half_width, closed):
        return Track(False, waypoints=points, closed=closed, half_width=half_width)

    def __setattr__(self, name, value):  # any public change invalidates the cached C view
        if not name.startswith("_"):
            object.__setattr__(self, "_c", None)
        object.__setattr__(self, name, value)

    def to_c(self):
        if getattr(self, "_c", None) is not None:
            return self._c
        t = A.TrackC()
        t.is_circle = int(self.is_circle)
        t.cx, t.cy = self.center
        t.radius = self.radius
        if self.waypoints is not None:
            t.n_waypoints = self.waypoints.shape[0]
            t.waypoints = A.dptr(self.waypoints)
        t.closed = int(self.closed)
        t.half_width = self.half_width
        self._c = t
        return t


def _obstacle_array(obstacles):
    if obstacles is None:
        return np.zeros((0, 3))
    rows = []
    for o in obstacles:
        if isinstance(o, CircleObstacle):
            rows.append([o.center[0], o.center[1], o.radius])
        else:
            rows.append(list(o))
    return _f64(rows, (-1, 3)) if rows else np.zeros((0, 3))


class TrackingTask:  # mppi.hpp:42-46
    """Task views are marshalled to C once per state: assigning any attribute (or the
    track's) rebuilds the view; edit obstacle arrays by re-assigning them, not in place."""
    kind = A.TASK_TRACKING

    def __init__(self, track: Track, v_desired: float, weights: TrackingWeights = None):
        self.track = track
        self.v_desired = v_desired
        self.weights = weights or TrackingWeights()
        self.obstacles = np.zeros((0, 3))
        self.goal = GoalSpec()
        self.avoidance = AvoidanceWeights()
        self.high_cost = 1e4

    def __setattr__(self, name, value):  # any public change invalidates the cached C view
        if not name.startswith("_"):
            object.__setattr__(self, "_c", None)
        object.__setattr__(self, name, value)

    def to_c(self):
        # the C view is built once per task state (plan_step's Python overhead was ~45 us
        # of re-marshalling the same task every tick); the track's own cache is checked too
        if getattr(self, "_c", None) is not None and (self.track is None or self.track._c is self._track_c):
            return self._c
        t = A.TaskC()
        t.kind = self.kind
        self._track_c = self.track.to_c() if self.track is not None else None
        if self._track_c is not None:
            t.track = C.pointer(self._track_c)
        t.v_desired = self.v_desired
        w = self.weights
        t.tracking = A.TrackingWeightsC(w.variance, w.deviation, w.slip, w.safety, w.speed)
        self._obs = _obstacle_array(self.obstacles)
        t.obstacles = A.dptr(self._obs) if self._obs.shape[0] else None
        t.n_obstacles = self._obs.shape[0]
        t.goal = (C.c_double * 3)(self.goal.position[0], self.goal.position[1],
                                  self.goal.capture_radius)
        a = self.avoidance
        t.avoidance = A.AvoidanceWeightsC(a.variance, a.obstacle, a.stage, a.terminal)
        t.high_cost = self.high_cost
        self._c = t
        return t


class AvoidanceTask(TrackingTask):  # mppi.hpp:47-52
    kind = A.TASK_AVOIDANCE

    def __init__(self, obstacles, goal: GoalSpec, weights: AvoidanceWeights = None,
                 high_cost: float = 1e4):
        super().__init__(None, 0.0)
        self.obstacles = obstacles
        self.goal = goal
        self.avoidance = weights or AvoidanceWeights()
        self.high_cost = high_cost


class CombinedTask(TrackingTask):
    """Path tracking + tightened obstacle chance constraints (BASELINE config 2).

    cost = tracking_cost (costs.cpp:127-149) + obstacle weight · Σ_k
    collision_indicator(x_{k+1}, obstacles, margins[k]) (costs.cpp:104-114),
    composed from unmodified reference terms."""
    kind = A.TASK_COMBINED

    def __init__(self, track: Track, v_desired: float, obstacles,
                 weights: TrackingWeights = None, obstacle_weight: float = 1.0):
        super().__init__(track, v_desired, weights)
        self.obstacles = obstacles
        self.avoidance = AvoidanceWeights(obstacle=obstacle_weight)


@dataclass
class StepDiagnostics:  # mppi.hpp:81-89
    best_cost: float = 0.0
    mean_cost: float = 0.0
    ess: float = 0.0
    weight_entropy: float = 0.0
    nonfinite_samples: int = 0
    tightening_infeasible: bool = False
    plan_ms: float = 0.0
    command_ms: float = 0.0


# ----------------------------------------------------------------- GP model
class GpModel:
    """Exact GP with device-resident factors (gp.hpp:30-98)."""

    def __init__(self, handle, device=0):
        self._h = handle
        self.device = device

    @staticmethod
    def fit(inputs, outputs, kernels, device: int = 0) -> "GpModel":
        X = _f64(inputs)
        if X.ndim != 2 or X.shape[1] != 4:
            raise ValueError("GpModel::fit: inputs must be n x 4 with n >= 1")
        Y = _f64(outputs)
        if Y.ndim == 1:
            Y = Y[:, None]
        if Y.shape[0] != X.shape[0]:
            raise ValueError("GpModel::fit: outputs must be n x m with m >= 1")
        rows = [k.as_row() if isinstance(k, KernelParams) else list(k) for k in kernels]
        if len(rows) != Y.shape[1]:
            raise ValueError("GpModel::fit: one KernelParams per output column required")
        K = _f64(rows, (-1, 6))
        h = C.c_void_p()
        A.check(A.lib().gpmppi_model_fit(A.dptr(X), A.dptr(Y), X.shape[0], Y.shape[1], A.dptr(K),
                                         device, C.byref(h)))
        return GpModel(h, device)

    @staticmethod
    def load(path: str, device: int = 0) -> "GpModel":
        h = C.c_void_p()
        A.check(A.lib().gpmppi_model_load(path.encode(), device, C.byref(h)))
        return GpModel(h, device)

    def save(self, path: str) -> None:
        A.check(A.lib().gpmppi_model_save(self._h, path.encode()))

    def __del__(self):
        if getattr(self, "_h", None) and A._LIB is not None:
            A._LIB.gpmppi_model_free(self._h)
            self._h = None

    @property
    def handle(self):
        return self._h

    @property
    def n_points(self) -> int:
        return A.lib().gpmppi_model_n_points(self._h)

    @property
    def n_outputs(self) -> int:
        return A.lib().gpmppi_model_n_outputs(self._h)

    def n_groups(self) -> int:
        return A.lib().gpmppi_model_n_groups(self._h)

    def group_jitter(self, g: int) -> float:
        return A.lib().gpmppi_model_group_jitter(self._h, g)

    def log_marginal_likelihood(self, output: int) -> float:
        return A.lib().gpmppi_model_log_marginal_likelihood(self._h, output)

    def training_data(self):
        X = np.empty((self.n_points, 4))
        Y = np.empty((self.n_points, self.n_outputs))
        A.check(A.lib().gpmppi_model_training_data(self._h, A.dptr(X), A.dptr(Y)))
        return X, Y

    def predict_batch(self, queries):
        Q = _f64(queries)
        if Q.ndim != 2 or Q.shape[1] != 4:
            raise ValueError("GpModel::predict_batch: queries must be S x 4")
        S, m = Q.shape[0], self.n_outputs
        mean = np.empty((S, m))
        var = np.empty((S, m))
        A.check(A.lib().gpmppi_model_predict_batch(self._h, A.dptr(Q), S, A.dptr(mean), A.dptr(var)))
        return mean, var

    def variance_batch(self, queries, path: int):
        """Per-group variance through a solve variance path (VAR_FFMA / VAR_TC_*)."""
        Q = _f64(queries, (-1, 4))
        out = np.empty((Q.shape[0], self.n_groups()))
        A.check(A.lib().gpmppi_model_variance_batch(self._h, A.dptr(Q), Q.shape[0], path,
                                                    A.dptr(out)))
        return out

    def predict(self, query):
        q = _f64(query, (1, 4))
        if not np.isfinite(q).all():
            raise ValueError("GpModel::predict: non-finite query")
        mean, var = self.predict_batch(q)
        return mean[0], var[0]


# ----------------------------------------------------------------- planner
@dataclass
class TrainedModels:  # harness.hpp:41-46
    has_gp: bool = False
    gp: Optional[GpModel] = None
    edd5: Edd5Params = field(default_factory=lambda: Edd5Params.ideal(0.37))
    nominal: NominalParams = field(default_factory=NominalParams)


def load_models(path: str, device: int = 0) -> TrainedModels:
    """Models file GPMPPIM1 (harness.cpp:264-284); the GP is refit on load as GpModel::load."""
    e, n, h = A.Edd5C(), A.NominalC(), C.c_void_p()
    A.check(A.lib().gpmppi_models_load(path.encode(), device, C.byref(e), C.byref(n), C.byref(h)))
    gp = GpModel(h, device) if h.value else None
    return TrainedModels(gp is not None, gp, Edd5Params(e.alpha_l, e.alpha_r, e.x_icr, e.y_icr_l, e.y_icr_r),
                         NominalParams(n.tau_v, n.tau_omega, n.dt))


def save_models(path: str, models: TrainedModels) -> None:
    """Models file GPMPPIM1 (harness.cpp:249-262)."""
    p = models.edd5
    e = A.Edd5C(p.alpha_l, p.alpha_r, p.x_icr, p.y_icr_l, p.y_icr_r)
    n = A.NominalC(models.nominal.tau_v, models.nominal.tau_omega, models.nominal.dt)
    gp = models.gp.handle if (models.has_gp and models.gp is not None) else None
    A.check(A.lib().gpmppi_models_save(path.encode(), C.byref(e), C.byref(n), gp))


class GpEnsemble:  # mppi.hpp:30-33
    def __init__(self, model: GpModel, n_terrains: int):
        self.model = model
        self.n_terrains = n_terrains


class Edd5Baseline:  # mppi.hpp:34-37
    def __init__(self, params: Edd5Params, track_width: float = 0.4):
        self.params = params
        self.track_width = track_width


class UnicycleBaseline:  # mppi.hpp:38
    pass


class NominalDynamic:
    """Dynamic unicycle with zero GP residual (BASELINE config 1 extension)."""


def _model_c(model):
    pm = A.PredictionModelC()
    if isinstance(model, GpEnsemble):
        pm.kind = A.MODEL_GP_ENSEMBLE
        pm.gp = model.model.handle
        pm.n_terrains = model.n_terrains
    elif isinstance(model, Edd5Baseline):
        pm.kind = A.MODEL_EDD5
        p = model.params
        pm.edd5 = A.Edd5C(p.alpha_l, p.alpha_r, p.x_icr, p.y_icr_l, p.y_icr_r)
        pm.track_width = model.track_width
    elif isinstance(model, UnicycleBaseline):
        pm.kind = A.MODEL_UNICYCLE
    elif isinstance(model, NominalDynamic):
        pm.kind = A.MODEL_NOMINAL
    else:
        raise ValueError("Planner: unknown prediction model")
    return pm


class Planner:
    """B200 GP-MPPI planner (mppi.hpp:96-143)."""

    def __init__(self, cfg: MppiConfig, model, nominal: NominalParams = None, p_x: float = 0.95,
                 device: int = 0):
        nominal = nominal or NominalParams()
        self.cfg = cfg
        self._model_ref = model  # keep the non-owning GP model alive
        self._cfg_c = cfg.to_c()
        self._pm_c = _model_c(model)
        self._nom_c = A.NominalC(nominal.tau_v, nominal.tau_omega, nominal.dt)
        h = C.c_void_p()
        A.check(A.lib().gpmppi_planner_create(C.byref(self._cfg_c), C.byref(self._pm_c),
                                              C.byref(self._nom_c), p_x, device, C.byref(h)))
        self._h = h
        self.T = cfg.horizon
        self.K = cfg.samples

    def __del__(self):
        if getattr(self, "_h", None) and A._LIB is not None:
            A._LIB.gpmppi_planner_free(self._h)
            self._h = None

    # -- Planner::plan_step (mppi.cpp:464-475)
    def plan_step(self, x0, task, diag: Optional[StepDiagnostics] = None):
        st = self.__dict__.get("_step_io")
        if st is None:  # per-planner call buffers and their C pointers, built once
            xb, cb, db = np.empty(5), np.empty(2), A.DiagC()
            st = (xb, A.dptr(xb), cb, A.dptr(cb), db, C.byref(db), A.lib().gpmppi_planner_plan_step)
            self.__dict__["_step_io"] = st
        xb, xp, cb, cp, d, dref, fn = st
        xb[:] = np.asarray(x0, dtype=np.float64).reshape(5)
        tc = task.to_c()
        A.check(fn(self._h, xp, C.byref(tc), cp, dref))
        cmd = cb.copy()
        if diag is not None:
            for k, _ in A.DiagC._fields_:
                setattr(diag, k, getattr(d, k))
            diag.tightening_infeasible = bool(d.tightening_infeasible)
        return cmd

    def set_terrain_weights(self, w):
        w = _f64(w, (-1,))
        A.check(A.lib().gpmppi_planner_set_terrain_weights(self._h, A.dptr(w), w.shape[0]))

    def terrain_weights(self):
        buf = np.empty(64)
        R = A.lib().gpmppi_planner_terrain_weights(self._h, A.dptr(buf))
        return buf[:R].copy()

    def nominal_sequence(self):
        s = np.empty((self.T, 2))
        A.check(A.lib().gpmppi_planner_nominal_sequence(self._h, A.dptr(s)))
        return s

    def set_nominal_sequence(self, seq):
        s = _f64(seq, (self.T, 2))
        A.check(A.lib().gpmppi_planner_set_nominal_sequence(self._h, A.dptr(s)))

    def horizon_covariances(self):
        c = np.empty((self.T, 5, 5))
        A.check(A.lib().gpmppi_planner_horizon_covariances(self._h, A.dptr(c)))
        return c

    def lane_radii(self):
        r = np.empty(self.T)
        n = A.lib().gpmppi_planner_lane_radii(self._h, A.dptr(r))
        if n < 0:
            A.check(A.CUDA_ERROR)
        return r[:n].copy()

    def obstacle_margins(self):
        m = np.empty(self.T * A.MAX_OBSTACLES)
        O = A.lib().gpmppi_planner_obstacle_margins(self._h, A.dptr(m))
        if O < 0:
            A.check(A.CUDA_ERROR)
        return m[: self.T * O].reshape(self.T, O).copy()

    def set_thresholds(self, r_bar=None, margins=None):
        r = None if r_bar is None else _f64(r_bar, (self.T,))
        m = None if margins is None else _f64(margins, (self.T, -1))
        O = 0 if m is None else m.shape[1]
        A.check(A.lib().gpmppi_planner_set_thresholds(self._h, A.dptr(r), A.dptr(m), O))

    def tick(self) -> int:
        return A.lib().gpmppi_planner_tick(self._h)

    def config(self) -> MppiConfig:
        return self.cfg

    # -- noise / parity hooks
    def set_noise_mode(self, mode: int):
        A.check(A.lib().gpmppi_planner_set_noise_mode(self._h, mode))

    def inject_noise(self, eps):
        e = _f64(eps, (self.samples_local(), self.T, 2))
        A.check(A.lib().gpmppi_planner_inject_noise(self._h, A.dptr(e)))

    def philox_noise(self, tick: int):
        e = np.empty((self.samples_local(), self.T, 2))
        A.check(A.lib().gpmppi_planner_philox_noise(self._h, tick, A.dptr(e)))
        return e

    def samples_local(self) -> int:
        return A.lib().gpmppi_planner_samples(self._h)

    def sample_costs(self):
        c = np.empty(self.samples_local())
        A.check(A.lib().gpmppi_planner_sample_costs(self._h, A.dptr(c)))
        return c

    def sample_weights(self):
        w = np.empty(self.samples_local())
        A.check(A.lib().gpmppi_planner_sample_weights(self._h, A.dptr(w)))
        return w

    def flags(self):
        K, T = self.samples_local(), self.T
        v = np.empty((K, T), np.uint8)
        c = np.empty((K, T), np.uint8)
        t = np.empty(K, np.uint8)
        a = np.empty(K, np.uint8)
        A.check(A.lib().gpmppi_planner_flags(self._h, A.u8ptr(v), A.u8ptr(c), A.u8ptr(t),
                                             A.u8ptr(a)))
        return dict(viol=v, coll=c, terminal=t, alive=a)

    def set_variance_path(self, path: int):
        A.check(A.lib().gpmppi_planner_set_variance_path(self._h, path))

    def variance_path(self) -> int:
        return A.lib().gpmppi_planner_variance_path(self._h)

    def bench_device(self, x0, task, ticks: int, flush_l2: bool = True):
        """Device-resident timing: per-tick CUDA-event ms and per-phase sums."""
        x = _f64(x0, (5,))
        tc = task.to_c()
        tick_ms = np.zeros(ticks)
        ph = np.zeros(4)
        A.check(A.lib().gpmppi_planner_bench_device(self._h, A.dptr(x), C.byref(tc), ticks,
                                                    int(flush_l2), A.dptr(tick_ms), A.dptr(ph)))
        return tick_ms, ph

    def io_bytes(self):
        h, d = C.c_int64(), C.c_int64()
        A.check(A.lib().gpmppi_planner_io_bytes(self._h, C.byref(h), C.byref(d)))
        return h.value, d.value

    # -- sharded solve
    def set_shard(self, begin: int, count: int):
        A.check(A.lib().gpmppi_planner_set_shard(self._h, begin, count))

    def plan_partial(self, x0, task, device_tuple_ptr: int):
        x = _f64(x0, (5,))
        tc = task.to_c()
        A.check(A.lib().gpmppi_planner_plan_partial(self._h, A.dptr(x), C.byref(tc),
                                                    C.c_void_p(device_tuple_ptr)))

    def attach_comm(self, unique_id: bytes, n_ranks: int, rank: int):
        """Shard this planner's samples over an NCCL communicator (collective: every rank
        calls it with the same id). plan_step then runs the sharded tick in the library."""
        buf = C.create_string_buffer(bytes(unique_id), 128)
        A.check(A.lib().gpmppi_planner_attach_comm(self._h, buf, n_ranks, rank))

    def shard(self):
        """(begin, count, n_ranks, rank) of this planner's global sample range."""
        b, c, n, r = C.c_int64(), C.c_int64(), C.c_int(), C.c_int()
        A.check(A.lib().gpmppi_planner_shard(self._h, C.byref(b), C.byref(c), C.byref(n), C.byref(r)))
        return b.value, c.value, n.value, r.value

    def set_command_first(self, on: bool = True):
        """plan_step returns at the command; the tightening pass completes behind it."""
        A.check(A.lib().gpmppi_planner_set_command_first(self._h, int(bool(on))))

    def wait_tightening(self, diag: Optional[StepDiagnostics] = None):
        """Wait for the last tick's tightening; completes its diagnostics (command-first mode)."""
        d = A.DiagC()
        A.check(A.lib().gpmppi_planner_wait_tightening(self._h, C.byref(d)))
        if diag is not None:
            for k, _ in A.DiagC._fields_:
                setattr(diag, k, getattr(d, k))
            diag.tightening_infeasible = bool(d.tightening_infeasible)
        return diag

    def plan_finish(self, device_tuples_ptr: int, n_ranks: int, diag=None):
        cmd = np.empty(2)
        d = A.DiagC()
        A.check(A.lib().gpmppi_planner_plan_finish(self._h, C.c_void_p(device_tuples_ptr), n_ranks,
                                                   A.dptr(cmd), C.byref(d)))
        if diag is not None:
            for k, _ in A.DiagC._fields_:
                setattr(diag, k, getattr(d, k))
        return cmd


class BatchPlanner(Planner):
    """B independent planners sharing one model (BASELINE config 4).

    Robot b is exactly ``Planner`` with ``cfg.seed = seeds[b]`` (default cfg.seed + b);
    all robots tick together through one launch sequence. Per-robot arrays are
    robot-major: ``plan_step(x0[B,5], tasks[B]) -> commands[B,2]``.
    """

    def __init__(self, cfg: MppiConfig, model, n_robots: int, nominal: NominalParams = None,
                 p_x: float = 0.95, seeds=None, device: int = 0):
        nominal = nominal or NominalParams()
        self.cfg = cfg
        self._model_ref = model
        self._cfg_c = cfg.to_c()
        self._pm_c = _model_c(model)
        self._nom_c = A.NominalC(nominal.tau_v, nominal.tau_omega, nominal.dt)
        sd = None
        if seeds is not None:
            sd = (C.c_uint64 * n_robots)(*[int(s) for s in seeds])
        h = C.c_void_p()
        A.check(A.lib().gpmppi_planner_create_batch(C.byref(self._cfg_c), C.byref(self._pm_c),
                                                    C.byref(self._nom_c), p_x, n_robots, sd, device,
                                                    C.byref(h)))
        self._h = h
        self.T = cfg.horizon
        self.K = cfg.samples
        self.B = n_robots

    def robots(self) -> int:
        return A.lib().gpmppi_planner_robots(self._h)

    def _tasks_c(self, tasks):
        if len(tasks) != self.B:
            raise ValueError("BatchPlanner: need one task per robot")
        arr = (A.TaskC * self.B)()
        keep = []  # to_c() rebinds the task's buffers: hold every copy until the call returns
        for b, t in enumerate(tasks):
            arr[b] = t.to_c()
            keep.append((t._track_c, t._obs))
        self._task_keep = keep
        return arr

    def plan_step(self, x0, tasks, diags=None):
        x = _f64(x0, (self.B, 5))
        tc = self._tasks_c(tasks)
        cmd = np.empty((self.B, 2))
        d = (A.DiagC * self.B)()
        A.check(A.lib().gpmppi_planner_plan_step_batch(self._h, A.dptr(x), tc, A.dptr(cmd), d))
        if diags is not None:
            for b in range(self.B):
                for k, _ in A.DiagC._fields_:
                    setattr(diags[b], k, getattr(d[b], k))
                diags[b].tightening_infeasible = bool(d[b].tightening_infeasible)
        return cmd

    def set_robot_terrain_weights(self, robot: int, w):
        w = _f64(w, (-1,))
        A.check(A.lib().gpmppi_planner_set_robot_terrain_weights(self._h, robot, A.dptr(w), w.shape[0]))

    def terrain_weights(self):
        buf = np.empty(self.B * A.MAX_TERRAINS)
        R = A.lib().gpmppi_planner_terrain_weights(self._h, A.dptr(buf))
        return buf[: self.B * R].reshape(self.B, R).copy()

    def nominal_sequence(self):
        s = np.empty((self.B, self.T, 2))
        A.check(A.lib().gpmppi_planner_nominal_sequence(self._h, A.dptr(s)))
        return s

    def set_nominal_sequence(self, seq):
        s = _f64(seq, (self.B, self.T, 2))
        A.check(A.lib().gpmppi_planner_set_nominal_sequence(self._h, A.dptr(s)))

    def horizon_covariances(self):
        c = np.empty((self.B, self.T, 5, 5))
        A.check(A.lib().gpmppi_planner_horizon_covariances(self._h, A.dptr(c)))
        return c

    def lane_radii(self):
        r = np.empty((self.B, self.T))
        n = A.lib().gpmppi_planner_lane_radii(self._h, A.dptr(r))
        if n < 0:
            A.check(A.CUDA_ERROR)
        return r if n else np.zeros((self.B, 0))

    def obstacle_margins(self):
        m = np.empty(self.B * self.T * A.MAX_OBSTACLES)
        O = A.lib().gpmppi_planner_obstacle_margins(self._h, A.dptr(m))
        if O < 0:
            A.check(A.CUDA_ERROR)
        return m[: self.B * self.T * O].reshape(self.B, self.T, O).copy()

    def set_thresholds(self, r_bar=None, margins=None):
        r = None if r_bar is None else _f64(r_bar, (self.B, self.T))
        m = None if margins is None else _f64(margins, (self.B, self.T, -1))
        O = 0 if m is None else m.shape[2]
        A.check(A.lib().gpmppi_planner_set_thresholds(self._h, A.dptr(r), A.dptr(m), O))

    def inject_noise(self, eps):
        e = _f64(eps, (self.B, self.samples_local(), self.T, 2))
        A.check(A.lib().gpmppi_planner_inject_noise(self._h, A.dptr(e)))

    def philox_noise(self, tick: int):
        e = np.empty((self.B, self.samples_local(), self.T, 2))
        A.check(A.lib().gpmppi_planner_philox_noise(self._h, tick, A.dptr(e)))
        return e

    def sample_costs(self):
        c = np.empty((self.B, self.samples_local()))
        A.check(A.lib().gpmppi_planner_sample_costs(self._h, A.dptr(c)))
        return c

    def sample_weights(self):
        w = np.empty((self.B, self.samples_local()))
        A.check(A.lib().gpmppi_planner_sample_weights(self._h, A.dptr(w)))
        return w

    def flags(self):
        B, K, T = self.B, self.samples_local(), self.T
        v = np.empty((B, K, T), np.uint8)
        c = np.empty((B, K, T), np.uint8)
        t = np.empty((B, K), np.uint8)
        a = np.empty((B, K), np.uint8)
        A.check(A.lib().gpmppi_planner_flags(self._h, A.u8ptr(v), A.u8ptr(c), A.u8ptr(t),
                                             A.u8ptr(a)))
        return dict(viol=v, coll=c, terminal=t, alive=a)

    def bench_device(self, x0, tasks, ticks: int, flush_l2: bool = True):
        x = _f64(x0, (self.B, 5))
        tc = self._tasks_c(tasks)
        tick_ms = np.zeros(ticks)
        ph = np.zeros(4)
        A.check(A.lib().gpmppi_planner_bench_device(self._h, A.dptr(x), tc, ticks, int(flush_l2),
                                                    A.dptr(tick_ms), A.dptr(ph)))
        return tick_ms, ph

    def set_shard(self, begin: int, count: int):
        raise ValueError("BatchPlanner: batched planners shard by robot, not by sample")


# ----------------------------------------------------------------- free functions
# Reference free functions (mppi.hpp:60-79), computed on the device.
@dataclass
class RolloutResult:  # mppi.hpp:53-56
    states: np.ndarray       # (T+1) x 5
    corrections: np.ndarray  # T x 4: mean_v, mean_w, var_v (cov 0,0), var_w (cov 1,1)


def rollout(x0, seq, model, weights=None, nominal: NominalParams = None, device: int = 0) -> RolloutResult:
    """Mean-only rollout of one control sequence (mppi.cpp:80-111)."""
    nominal = nominal or NominalParams()
    x = _f64(x0, (5,))
    sq = _f64(seq, (-1, 2))
    T = sq.shape[0]
    R = model.n_terrains if isinstance(model, GpEnsemble) else 0
    w = _f64(weights if weights is not None else np.full(max(R, 1), 1.0 / max(R, 1)), (-1,))
    states, corr = np.empty((T + 1, 5)), np.empty((T, 4))
    pm = _model_c(model)
    nom = A.NominalC(nominal.tau_v, nominal.tau_omega, nominal.dt)
    A.check(A.lib().gpmppi_rollout(C.byref(pm), C.byref(nom), A.dptr(w), w.shape[0] if R else 0,
                                   A.dptr(x), A.dptr(sq), T, device, A.dptr(states), A.dptr(corr)))
    return RolloutResult(states, corr)


def sample_perturbations(cfg: MppiConfig, tick: int, device: int = 0):
    """K x T x 2 Gaussian perturbations (mppi.cpp:113-123), Philox sampler keyed by (seed, tick, s)."""
    c = cfg.to_c()
    eps = np.empty((cfg.samples, cfg.horizon, 2))
    A.check(A.lib().gpmppi_sample_perturbations(C.byref(c), tick, device, A.dptr(eps)))
    return eps


def trajectory_weights(costs, lam: float, device: int = 0):
    """Softmax weights with a min-cost baseline (mppi.cpp:125-145)."""
    c = _f64(costs, (-1,))
    w = np.empty_like(c)
    A.check(A.lib().gpmppi_trajectory_weights(A.dptr(c), c.shape[0], lam, device, A.dptr(w)))
    return w


def update_controls(nominal, eps, weights, bounds: ControlBounds = None, device: int = 0):
    """Perturbation-weighted update, clamped (mppi.cpp:147-164)."""
    bounds = bounds or ControlBounds()
    nom = _f64(nominal, (-1, 2))
    e = _f64(eps, (-1, nom.shape[0], 2))
    w = _f64(weights, (-1,))
    if e.shape[0] != w.shape[0]:
        raise ValueError("update_controls: one weight per sample required")
    out = np.empty_like(nom)
    lo, hi = _f64(bounds.lo), _f64(bounds.hi)
    A.check(A.lib().gpmppi_update_controls(A.dptr(nom), nom.shape[0], A.dptr(e), A.dptr(w), w.shape[0],
                                           A.dptr(lo), A.dptr(hi), device, A.dptr(out)))
    return out


def shift_horizon(seq, device: int = 0):
    """Drop the first control, repeat the last (mppi.cpp:166-173)."""
    s = _f64(seq, (-1, 2))
    out = np.empty_like(s)
    A.check(A.lib().gpmppi_shift_horizon(A.dptr(s), s.shape[0], device, A.dptr(out)))
    return out


def shard_range(total: int, world: int, rank: int):
    """Contiguous global sample range of `rank`: [begin, begin+count)."""
    base, extra = divmod(total, world)
    begin = rank * base + min(rank, extra)
    return begin, base + (1 if rank < extra else 0)


def apply_tuple(tup, nominal, lo=(-0.5, -2.0), hi=(2.0, 2.0)):
    """Update + clamp + shift from a combined tuple (mppi.cpp:147-173), host arithmetic
    for the CPU multi-rank tests (the device runs the same in finish_kernel)."""
    T = len(nominal)
    Z = tup[1]
    dv = tup[6:].reshape(T, 2) / Z if Z > 0 else np.zeros((T, 2))
    upd = np.clip(np.asarray(nominal) + dv, lo, hi)
    return upd[0].copy(), np.vstack([upd[1:], upd[-1:]])


def nccl_unique_id() -> bytes:
    """A fresh ncclUniqueId (128 bytes) for Planner.attach_comm; broadcast it to every rank."""
    buf = C.create_string_buffer(128)
    A.check(A.lib().gpmppi_nccl_unique_id(buf))
    return buf.raw


def tuple_doubles(horizon: int) -> int:
    return A.lib().gpmppi_tuple_doubles(horizon)


def combine_tuples(tuples, horizon: int, lam: float):
    """Host restatement of the device tuple combine (for CPU multi-rank tests)."""
    t = _f64(tuples, (-1, tuple_doubles(horizon)))
    out = np.empty(t.shape[1])
    A.check(A.lib().gpmppi_combine_tuples_host(A.dptr(t), t.shape[0], horizon, lam, A.dptr(out)))
    return out


def flush_l2(device: int = 0) -> None:
    A.check(A.lib().gpmppi_flush_l2(device))


def kernel_launches() -> int:
    return A.lib().gpmppi_kernel_launches()


# ----------------------------------------------------------------- small host math
def chi2_quantile_2dof(p: float) -> float:  # uncertainty.cpp:8-13
    if not (p >= 0.0) or p >= 1.0:
        raise ValueError("chi2_quantile_2dof: p must lie in [0, 1)")
    return -2.0 * math.log1p(-p)
