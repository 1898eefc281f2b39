"""ctypes binding of the FP64 CPU oracle (oracle/gpmppi_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
CPU-baseline / reference legs of bench.py. The product package never imports
this module.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

ORC_MODEL_GP, ORC_MODEL_EDD5, ORC_MODEL_UNICYCLE, ORC_MODEL_NOMINAL = 0, 1, 2, 3
ORC_TASK_TRACKING, ORC_TASK_AVOIDANCE, ORC_TASK_COMBINED = 0, 1, 2

_dp = C.POINTER(C.c_double)
_u8p = C.POINTER(C.c_uint8)


class OracleError(Exception):
    pass


def _ptr(a):
    return a.ctypes.data_as(_dp) if a is not None else None


class Nominal(C.Structure):
    _fields_ = [("tau_v", C.c_double), ("tau_omega", C.c_double), ("dt", C.c_double)]


class Edd5(C.Structure):
    _fields_ = [(k, C.c_double) for k in ("alpha_l", "alpha_r", "x_icr", "y_icr_l", "y_icr_r")]


class Track(C.Structure):
    _fields_ = [
        ("is_circle", C.c_int),
        ("cx", C.c_double),
        ("cy", C.c_double),
        ("radius", C.c_double),
        ("n_waypoints", C.c_int),
        ("waypoints", _dp),
        ("closed", C.c_int),
        ("half_width", C.c_double),
    ]


class TrackingWeights(C.Structure):
    _fields_ = [(k, C.c_double) for k in ("variance", "deviation", "slip", "safety", "speed")]


class AvoidanceWeights(C.Structure):
    _fields_ = [(k, C.c_double) for k in ("variance", "obstacle", "stage", "terminal")]


class MppiConfig(C.Structure):
    _fields_ = [
        ("samples", C.c_int),
        ("horizon", C.c_int),
        ("lam", C.c_double),
        ("sigma_v2", C.c_double),
        ("sigma_w2", C.c_double),
        ("lo", C.c_double * 2),
        ("hi", C.c_double * 2),
        ("seed", C.c_uint64),
        ("threads", C.c_int),
    ]


class Task(C.Structure):
    _fields_ = [
        ("kind", C.c_int),
        ("track", C.POINTER(Track)),
        ("v_desired", C.c_double),
        ("tw", TrackingWeights),
        ("obstacles", _dp),
        ("n_obstacles", C.c_int),
        ("goal", C.c_double * 3),
        ("aw", AvoidanceWeights),
        ("high_cost", C.c_double),
    ]


class Diag(C.Structure):
    _fields_ = [
        ("best_cost", C.c_double),
        ("mean_cost", C.c_double),
        ("ess", C.c_double),
        ("weight_entropy", C.c_double),
        ("nonfinite_samples", C.c_int),
        ("tightening_infeasible", C.c_int),
        ("plan_ms", C.c_double),
    ]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


def blas_library():
    """(path, symbol prefix) of the optimised CBLAS bundled with scipy (OpenBLAS), or None."""
    try:
        import glob

        import scipy
        libs = sorted(glob.glob(os.path.join(os.path.dirname(scipy.__file__), "..", "scipy.libs",
                                             "libscipy_openblas-*.so")))
        return (os.path.realpath(libs[0]), "scipy_") if libs else None
    except Exception:
        return None


def use_blas(on: bool = True, native: bool = None) -> str:
    """Timed CPU baseline only: OpenBLAS GEMM/TRMM in place of Eigen's (gp.cpp:178-185).
    Returns a description of what is in use."""
    L = lib(native)
    if not on:
        L.orc_use_blas(None, None)
        return "scalar loops"
    b = blas_library()
    if b is None or L.orc_use_blas(b[0].encode(), b[1].encode()) != 0:
        L.orc_use_blas(None, None)
        return "scalar loops (OpenBLAS not found)"
    return "OpenBLAS " + os.path.basename(b[0])


def build(native: bool = False) -> str:
    target = "liboracle_native.so" if native else "liboracle.so"
    subprocess.run(["make", "-s", "-C", _HERE, "native" if native else "all"], check=True)
    return os.path.join(_HERE, target)


def lib(native: bool = None):
    """The oracle library. native=None follows GPMPPI_ORACLE_NATIVE=1 (the bench's timed
    CPU arm builds and loads a -march=native copy on the host that runs it)."""
    global _LIB
    if native is None:
        native = os.environ.get("GPMPPI_ORACLE_NATIVE") == "1"
    if _LIB is not None:
        return _LIB
    path = os.path.join(_HERE, "liboracle_native.so" if native else "liboracle.so")
    src = os.path.join(_HERE, "gpmppi_oracle.c")
    if not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(src):
        build(native)
    L = C.CDLL(path)
    L.orc_last_error.restype = C.c_char_p
    L.orc_splitmix64.restype = C.c_uint64
    L.orc_splitmix64.argtypes = [C.c_uint64]
    L.orc_derive_seed.restype = C.c_uint64
    L.orc_derive_seed.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
    L.orc_uniform_stream.argtypes = [C.c_uint64, C.c_int, _dp]
    L.orc_gaussian_stream.argtypes = [C.c_uint64, C.c_int, _dp]
    L.orc_sample_perturbations.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_uint64,
                                           C.c_uint64, _dp]
    for f in ("orc_wrap_angle", "orc_chi2_quantile_2dof", "orc_normal_cdf", "orc_normal_quantile"):
        getattr(L, f).restype = C.c_double
        getattr(L, f).argtypes = [C.c_double]
    L.orc_use_blas.argtypes = [C.c_char_p, C.c_char_p]
    L.orc_kernel_eval.restype = C.c_double
    L.orc_kernel_eval.argtypes = [_dp, _dp, _dp]
    L.orc_gp_fit.argtypes = [_dp, _dp, C.c_int, C.c_int, _dp, C.POINTER(C.c_void_p)]
    L.orc_gp_free.argtypes = [C.c_void_p]
    L.orc_gp_predict_batch.argtypes = [C.c_void_p, _dp, C.c_int, _dp, _dp]
    for f in ("orc_gp_n_points", "orc_gp_n_outputs", "orc_gp_n_groups"):
        getattr(L, f).argtypes = [C.c_void_p]
    L.orc_gp_group_jitter.restype = C.c_double
    L.orc_gp_group_jitter.argtypes = [C.c_void_p, C.c_int]
    L.orc_gp_lml.restype = C.c_double
    L.orc_gp_lml.argtypes = [C.c_void_p, C.c_int]
    L.orc_gp_group_export.argtypes = [C.c_void_p, C.c_int, _dp, _dp, _dp, _dp,
                                      C.POINTER(C.c_int), C.POINTER(C.c_int), _dp]
    L.orc_ensemble_combine.argtypes = [_dp, _dp, _dp, C.c_int, _dp, _dp]
    L.orc_step_nominal.argtypes = [_dp, _dp, C.POINTER(Nominal), _dp]
    L.orc_jacobian_nominal.argtypes = [_dp, _dp, C.POINTER(Nominal), _dp]
    L.orc_step_kinematic.argtypes = [_dp, _dp, C.c_double, _dp]
    L.orc_step_edd5.argtypes = [_dp, _dp, C.POINTER(Edd5), C.c_double, C.c_double, _dp]
    L.orc_lambda_max_2x2.restype = C.c_double
    L.orc_lambda_max_2x2.argtypes = [_dp]
    L.orc_propagate_belief.argtypes = [_dp, _dp, _dp, _dp, _dp, C.POINTER(Nominal), _dp, _dp]
    L.orc_tighten_lane_radius.restype = C.c_double
    L.orc_tighten_lane_radius.argtypes = [C.c_double, _dp, C.c_double]
    L.orc_tighten_obstacle_distance.restype = C.c_double
    L.orc_tighten_obstacle_distance.argtypes = [_dp, _dp, C.c_double, _dp, C.c_double, _dp, _dp,
                                                C.POINTER(C.c_int)]
    L.orc_centerline_distance.restype = C.c_double
    L.orc_centerline_distance.argtypes = [C.POINTER(Track), C.c_double, C.c_double]
    L.orc_slip_ratio.restype = C.c_double
    L.orc_slip_ratio.argtypes = [_dp, _dp]
    L.orc_collision_indicator.restype = C.c_double
    L.orc_collision_indicator.argtypes = [C.c_double, C.c_double, _dp, C.c_int, _dp]
    L.orc_tracking_cost.restype = C.c_double
    L.orc_tracking_cost.argtypes = [_dp, _dp, C.c_int, C.POINTER(Track), _dp, C.c_double, _dp,
                                    C.POINTER(TrackingWeights)]
    L.orc_avoidance_cost.restype = C.c_double
    L.orc_avoidance_cost.argtypes = [_dp, _dp, C.c_int, _dp, C.c_int, _dp, _dp,
                                     C.POINTER(AvoidanceWeights), C.c_double]
    L.orc_trajectory_weights.argtypes = [_dp, C.c_int, C.c_double, _dp]
    L.orc_update_controls.argtypes = [_dp, _dp, _dp, C.c_int, C.c_int, _dp, _dp, _dp]
    L.orc_shift_horizon.argtypes = [_dp, C.c_int, _dp]
    L.orc_rollout.argtypes = [C.c_int, C.c_void_p, C.c_int, _dp, C.POINTER(Nominal), C.POINTER(Edd5),
                              C.c_double, _dp, _dp, C.c_int, _dp, _dp]
    L.orc_planner_create.argtypes = [C.POINTER(MppiConfig), C.c_int, C.c_void_p, C.c_int,
                                     C.POINTER(Edd5), C.c_double, C.POINTER(Nominal), C.c_double,
                                     C.POINTER(C.c_void_p)]
    L.orc_planner_free.argtypes = [C.c_void_p]
    L.orc_planner_set_terrain_weights.argtypes = [C.c_void_p, _dp, C.c_int]
    L.orc_planner_plan_step.argtypes = [C.c_void_p, _dp, C.POINTER(Task), _dp, _dp,
                                        C.POINTER(Diag)]
    L.orc_planner_last_costs.argtypes = [C.c_void_p, _dp]
    L.orc_planner_last_weights.argtypes = [C.c_void_p, _dp]
    L.orc_planner_last_flags.argtypes = [C.c_void_p, _u8p, _u8p, _u8p, _u8p]
    L.orc_planner_nominal_sequence.argtypes = [C.c_void_p, _dp]
    L.orc_planner_horizon_covariances.argtypes = [C.c_void_p, _dp]
    L.orc_planner_lane_radii.argtypes = [C.c_void_p, _dp]
    L.orc_planner_obstacle_margins.argtypes = [C.c_void_p, _dp]
    L.orc_planner_tick.restype = C.c_uint64
    L.orc_planner_tick.argtypes = [C.c_void_p]
    L.orc_planner_set_nominal_sequence.argtypes = [C.c_void_p, _dp]
    L.orc_planner_set_thresholds.argtypes = [C.c_void_p, _dp, _dp, C.c_int]
    L.orc_rollout_threads_used.argtypes = [C.c_void_p]
    _LIB = L
    return L


def _check(rc):
    if rc != 0:
        msg = lib().orc_last_error().decode()
        if rc == 1:
            raise ValueError(msg)
        raise RuntimeError(msg)


def f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def sample_perturbations(K, T, sigma_sim, seed, tick):
    eps = np.empty((K, T, 2))
    lib().orc_sample_perturbations(K, T, sigma_sim[0], sigma_sim[1], seed, tick, _ptr(eps))
    return eps


def trajectory_weights(costs, lam):  # mppi.cpp:125-145
    c = f64(costs)
    w = np.empty_like(c)
    lib().orc_trajectory_weights(_ptr(c), c.shape[0], lam, _ptr(w))
    return w


def update_controls(nominal, eps, w, lo=(-0.5, -2.0), hi=(2.0, 2.0)):  # mppi.cpp:147-164
    nom, e, ww = f64(nominal), f64(eps), f64(w)
    out = np.empty_like(nom)
    lib().orc_update_controls(_ptr(nom), _ptr(e), _ptr(ww), e.shape[0], nom.shape[0],
                              _ptr(f64(lo)), _ptr(f64(hi)), _ptr(out))
    return out


def shift_horizon(seq):  # mppi.cpp:166-173
    s = f64(seq)
    out = np.empty_like(s)
    lib().orc_shift_horizon(_ptr(s), s.shape[0], _ptr(out))
    return out


def rollout(x0, seq, kind=ORC_MODEL_GP, gp=None, R=0, w=None, nominal=(0.5, 0.35, 0.05),
            edd5=(1.0, 1.0, 0.0, -0.2, 0.2), track_width=0.4):
    """mppi.cpp:80-111: (states (T+1)x5, corrections Tx4 = mean_v, mean_w, var_v, var_w)."""
    sq = f64(seq).reshape(-1, 2)
    T = sq.shape[0]
    states = np.empty((T + 1, 5))
    corr = np.empty((T, 4))
    ww = f64(w if w is not None else np.full(max(R, 1), 1.0 / max(R, 1)))
    _check(lib().orc_rollout(kind, gp.h if gp is not None else None, R, _ptr(ww), Nominal(*nominal),
                             Edd5(*edd5), track_width, _ptr(f64(x0)), _ptr(sq), T, _ptr(states),
                             _ptr(corr)))
    return states, corr


class GP:
    """Oracle GpModel (gp.cpp:61-198)."""

    def __init__(self, inputs, outputs, kernels):
        self.inputs = f64(inputs)
        self.outputs = f64(outputs)
        if self.outputs.ndim == 1:
            self.outputs = self.outputs[:, None]
        self.kernels = f64(kernels).reshape(-1, 6)
        h = C.c_void_p()
        n, m = self.inputs.shape[0], self.outputs.shape[1]
        _check(lib().orc_gp_fit(_ptr(self.inputs), _ptr(self.outputs), n, m,
                                _ptr(self.kernels), C.byref(h)))
        self.h = h
        self.n, self.m = n, m

    def __del__(self):
        if getattr(self, "h", None) and _LIB is not None:
            _LIB.orc_gp_free(self.h)
            self.h = None

    def predict_batch(self, q):
        q = f64(q).reshape(-1, 4)
        mean = np.empty((q.shape[0], self.m))
        var = np.empty((q.shape[0], self.m))
        _check(lib().orc_gp_predict_batch(self.h, _ptr(q), q.shape[0], _ptr(mean), _ptr(var)))
        return mean, var

    def n_groups(self):
        return lib().orc_gp_n_groups(self.h)

    def jitter(self, g=0):
        return lib().orc_gp_group_jitter(self.h, g)

    def lml(self, o):
        return lib().orc_gp_lml(self.h, o)

    def group(self, g=0):
        n = self.n
        ilt = np.empty((n, n))
        chol = np.empty((n, n))
        nout = C.c_int()
        outs = (C.c_int * 64)()
        k6 = np.empty(6)
        alphas = np.empty((n, self.m))
        aug = np.empty((n, 6))
        lib().orc_gp_group_export(self.h, g, _ptr(ilt), _ptr(chol), _ptr(alphas), _ptr(aug),
                                  outs, C.byref(nout), _ptr(k6))
        no = nout.value
        return dict(inv_lower_t=ilt, chol=chol, alphas=alphas[:, :no].copy(), inputs_aug=aug,
                    outputs=list(outs[:no]), kernel=k6)


def make_track(kind="circle", center=(0.0, 0.0), radius=2.0, half_width=0.4, waypoints=None,
               closed=True):
    t = Track()
    keep = None
    if kind == "circle":
        t.is_circle = 1
        t.cx, t.cy = center
        t.radius = radius
    else:
        keep = f64(waypoints).reshape(-1, 2)
        t.is_circle = 0
        t.n_waypoints = keep.shape[0]
        t.waypoints = _ptr(keep)
        t.closed = int(closed)
    t.half_width = half_width
    t._keep = keep
    return t


class Planner:
    """Oracle Planner (mppi.hpp:96-143) with parity outputs."""

    def __init__(self, samples, horizon, model_kind=ORC_MODEL_GP, gp=None, n_terrains=0,
                 lam=0.1, sigma_sim=(0.09, 0.25), lo=(-0.5, -2.0), hi=(2.0, 2.0), seed=0,
                 threads=0, nominal=(0.5, 0.35, 0.05), p_x=0.95, edd5=None, track_width=0.4,
                 native=None):
        self.L = lib(native)
        self.cfg = MppiConfig(samples, horizon, lam, sigma_sim[0], sigma_sim[1],
                              (C.c_double * 2)(*lo), (C.c_double * 2)(*hi), seed, threads)
        self.nominal = Nominal(*nominal)
        self.gp = gp
        e = Edd5(*(edd5 if edd5 is not None else (1.0, 1.0, 0.0, -0.2, 0.2)))
        h = C.c_void_p()
        rc = self.L.orc_planner_create(C.byref(self.cfg), model_kind, gp.h if gp else None,
                                       n_terrains, C.byref(e), track_width,
                                       C.byref(self.nominal), p_x, C.byref(h))
        _check(rc)
        self.h = h
        self.K, self.T = samples, horizon

    def __del__(self):
        if getattr(self, "h", None):
            self.L.orc_planner_free(self.h)
            self.h = None

    def set_terrain_weights(self, w):
        w = f64(w)
        _check(self.L.orc_planner_set_terrain_weights(self.h, _ptr(w), w.shape[0]))

    def plan_step(self, x0, task, eps=None):
        x0 = f64(x0)
        cmd = np.empty(2)
        d = Diag()
        e = f64(eps) if eps is not None else None
        _check(self.L.orc_planner_plan_step(self.h, _ptr(x0), C.byref(task), _ptr(e), _ptr(cmd),
                                            C.byref(d)))
        return cmd, d.as_dict()

    def costs(self):
        c = np.empty(self.K)
        self.L.orc_planner_last_costs(self.h, _ptr(c))
        return c

    def weights(self):
        w = np.empty(self.K)
        self.L.orc_planner_last_weights(self.h, _ptr(w))
        return w

    def flags(self):
        v = np.empty((self.K, self.T), np.uint8)
        c = np.empty((self.K, self.T), np.uint8)
        t = np.empty(self.K, np.uint8)
        a = np.empty(self.K, np.uint8)
        u8 = lambda x: x.ctypes.data_as(_u8p)  # noqa: E731
        self.L.orc_planner_last_flags(self.h, u8(v), u8(c), u8(t), u8(a))
        return dict(viol=v, coll=c, terminal=t, alive=a)

    def nominal_sequence(self):
        s = np.empty((self.T, 2))
        self.L.orc_planner_nominal_sequence(self.h, _ptr(s))
        return s

    def set_nominal_sequence(self, seq):
        seq = f64(seq)
        self.L.orc_planner_set_nominal_sequence(self.h, _ptr(seq))

    def horizon_covariances(self):
        c = np.empty((self.T, 5, 5))
        self.L.orc_planner_horizon_covariances(self.h, _ptr(c))
        return c

    def lane_radii(self):
        r = np.empty(self.T)
        self.L.orc_planner_lane_radii(self.h, _ptr(r))
        return r

    def obstacle_margins(self):
        O = self.L.orc_planner_obstacle_margins(self.h, None)
        m = np.empty((self.T, max(O, 0)))
        if O > 0:
            self.L.orc_planner_obstacle_margins(self.h, _ptr(m))
        return m

    def tick(self):
        return self.L.orc_planner_tick(self.h)

    def threads_used(self):
        return self.L.orc_rollout_threads_used(self.h)


def make_task(kind, track=None, v_desired=2.0, tracking_weights=(0.1, 1.0, 0.3, 1.0, 0.2),
              obstacles=None, goal=(8.0, 0.0, 0.5), avoidance_weights=(0.1, 1.0, 0.5, 1.0),
              high_cost=1e4):
    t = Task()
    t.kind = kind
    if track is not None:
        t.track = C.pointer(track)
    t.v_desired = v_desired
    t.tw = TrackingWeights(*tracking_weights)
    obs = f64(obstacles).reshape(-1, 3) if obstacles is not None else np.zeros((0, 3))
    t.obstacles = _ptr(obs) if obs.shape[0] else None
    t.n_obstacles = obs.shape[0]
    t.goal = (C.c_double * 3)(*goal)
    t.aw = AvoidanceWeights(*avoidance_weights)
    t.high_cost = high_cost
    t._keep = (obs, track)
    return t


def select_kernel_grid(inputs, outputs):
    """CPU restatement of select_kernel_grid (gp.cpp:274-366): numpy Cholesky per cell,
    the reference's sweep order and strict-greater argmax. Returns (sv, lengthscales, nv, lml).
    Checker for the device grid (tests only)."""
    X = np.asarray(inputs, dtype=np.float64)
    Y = np.asarray(outputs, dtype=np.float64)
    n, m = X.shape[0], Y.shape[1]
    if n < 2:
        raise ValueError("select_kernel_grid: need at least 2 points")
    base = np.maximum(np.sqrt(((X - X.mean(0)) ** 2).sum(0) / (n - 1)), 1e-3)
    pooled = max(float(sum(((Y[:, j] - Y[:, j].mean()) ** 2).sum() / (n - 1) for j in range(m))) / m,
                 1e-10)
    S = X / base
    sq = (S * S).sum(1)
    d2 = -2.0 * S @ S.T + sq[:, None] + sq[None, :]
    d2 = np.maximum(0.5 * (d2 + d2.T), 0.0)
    log2pi = math.log(2.0 * math.pi)

    def score(sv, scale, nv):
        K = sv * np.exp(-d2 / (2.0 * scale * scale))
        K[np.diag_indices(n)] += nv
        try:
            L = np.linalg.cholesky(K)
        except np.linalg.LinAlgError:
            return -math.inf
        logdet = float(np.log(np.diag(L)).sum())
        A = np.linalg.solve(L.T, np.linalg.solve(L, Y))
        return float(sum(-0.5 * Y[:, j] @ A[:, j] - logdet - 0.5 * n * log2pi for j in range(m)))

    def logspace(lo, hi, k):
        return [10.0 ** (lo + (hi - lo) * (0.0 if k == 1 else i / (k - 1))) for i in range(k)]

    best = [-math.inf, pooled, 1.0, pooled * 0.1]

    def sweep(svs, ss, nvs):
        for sv in svs:
            for s in ss:
                for nv in nvs:
                    val = score(sv, s, nv)
                    if val > best[0]:
                        best[:] = [val, sv, s, nv]

    sweep([pooled * f for f in logspace(-1.5, 1.5, 5)], logspace(-1.0, 1.0, 7),
          [pooled * f for f in logspace(-3.0, 0.5, 5)])
    sv0, s0, nv0 = best[1], best[2], best[3]
    sweep([sv0 * f for f in logspace(-0.5, 0.5, 5)], [s0 * f for f in logspace(-0.35, 0.35, 7)],
          [nv0 * f for f in logspace(-0.6, 0.6, 5)])
    return best[1], tuple(float(b * best[2]) for b in base), best[3], best[0]


