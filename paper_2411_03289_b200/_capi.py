"""ctypes binding of include/gpmppi_b200.h (lib/libgpmppi_b200.so).

The library is the product: every compute call runs sm_100a kernels. If the
shared object is missing or cannot be loaded this module raises — there is no
CPU fallback anywhere in the package.
"""
from __future__ import annotations

import ctypes as C
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
# GPMPPI_LIB selects an in-tree A/B experiment build (lib/libgpmppi_b200_<variant>.so)
LIB_PATH = os.environ.get("GPMPPI_LIB") or os.path.join(_PKG, "lib", "libgpmppi_b200.so")

_dp = C.POINTER(C.c_double)
_u8p = C.POINTER(C.c_uint8)
_vp = C.c_void_p

OK, INVALID_ARGUMENT, RUNTIME_ERROR, LOGIC_ERROR, CUDA_ERROR = 0, 1, 2, 3, 4
MODEL_GP_ENSEMBLE, MODEL_EDD5, MODEL_UNICYCLE, MODEL_NOMINAL = 0, 1, 2, 3
TASK_TRACKING, TASK_AVOIDANCE, TASK_COMBINED = 0, 1, 2
NOISE_PHILOX, NOISE_INJECTED = 0, 1
VAR_FFMA, VAR_TC_3XTF32, VAR_TC_1XTF32, VAR_TC_3XF16, VAR_TC_3XF16_PAIR = 0, 1, 2, 3, 4
MAX_WAYPOINTS = 64
MAX_OBSTACLES = 64
MAX_TERRAINS = 16


class CudaError(RuntimeError):
    """No usable CUDA device, or a kernel launch failed."""


class MppiConfigC(C.Structure):
    _fields_ = [("samples", C.c_int), ("horizon", C.c_int), ("lam", C.c_double),
                ("sigma_v2", C.c_double), ("sigma_w2", C.c_double), ("lo", C.c_double * 2),
                ("hi", C.c_double * 2), ("seed", C.c_uint64), ("threads", C.c_int)]


class NominalC(C.Structure):
    _fields_ = [("tau_v", C.c_double), ("tau_omega", C.c_double), ("dt", C.c_double)]


class Edd5C(C.Structure):
    _fields_ = [(k, C.c_double) for k in ("alpha_l", "alpha_r", "x_icr", "y_icr_l", "y_icr_r")]


class PredictionModelC(C.Structure):
    _fields_ = [("kind", C.c_int), ("gp", _vp), ("n_terrains", C.c_int), ("edd5", Edd5C),
                ("track_width", C.c_double)]


class TrackC(C.Structure):
    _fields_ = [("is_circle", C.c_int), ("cx", C.c_double), ("cy", C.c_double),
                ("radius", C.c_double), ("n_waypoints", C.c_int), ("waypoints", _dp),
                ("closed", C.c_int), ("half_width", C.c_double)]


class TrackingWeightsC(C.Structure):
    _fields_ = [(k, C.c_double) for k in ("variance", "deviation", "slip", "safety", "speed")]


class AvoidanceWeightsC(C.Structure):
    _fields_ = [(k, C.c_double) for k in ("variance", "obstacle", "stage", "terminal")]


class TaskC(C.Structure):
    _fields_ = [("kind", C.c_int), ("track", C.POINTER(TrackC)), ("v_desired", C.c_double),
                ("tracking", TrackingWeightsC), ("obstacles", _dp), ("n_obstacles", C.c_int),
                ("goal", C.c_double * 3), ("avoidance", AvoidanceWeightsC),
                ("high_cost", C.c_double)]


class DiagC(C.Structure):
    _fields_ = [("best_cost", C.c_double), ("mean_cost", C.c_double), ("ess", C.c_double),
                ("weight_entropy", C.c_double), ("nonfinite_samples", C.c_int),
                ("tightening_infeasible", C.c_int), ("plan_ms", C.c_double),
                ("command_ms", C.c_double)]


_LIB = None

# (name, restype, argtypes) for every symbol include/gpmppi_b200.h declares
SIGNATURES = [
    ("gpmppi_last_error", C.c_char_p, []),
    ("gpmppi_abi_version", C.c_int, []),
    ("gpmppi_kernel_launches", C.c_uint64, []),
    ("gpmppi_model_fit", C.c_int, [_dp, _dp, C.c_int64, C.c_int64, _dp, C.c_int, C.POINTER(_vp)]),
    ("gpmppi_model_load", C.c_int, [C.c_char_p, C.c_int, C.POINTER(_vp)]),
    ("gpmppi_model_save", C.c_int, [_vp, C.c_char_p]),
    ("gpmppi_models_load", C.c_int, [C.c_char_p, C.c_int, C.POINTER(Edd5C), C.POINTER(NominalC), C.POINTER(_vp)]),
    ("gpmppi_models_save", C.c_int, [C.c_char_p, C.POINTER(Edd5C), C.POINTER(NominalC), _vp]),
    ("gpmppi_model_free", None, [_vp]),
    ("gpmppi_model_n_points", C.c_int, [_vp]),
    ("gpmppi_model_n_outputs", C.c_int, [_vp]),
    ("gpmppi_model_n_groups", C.c_int, [_vp]),
    ("gpmppi_model_group_jitter", C.c_double, [_vp, C.c_int]),
    ("gpmppi_model_log_marginal_likelihood", C.c_double, [_vp, C.c_int]),
    ("gpmppi_model_training_data", C.c_int, [_vp, _dp, _dp]),
    ("gpmppi_model_predict_batch", C.c_int, [_vp, _dp, C.c_int64, _dp, _dp]),
    ("gpmppi_model_variance_batch", C.c_int, [_vp, _dp, C.c_int64, C.c_int, _dp]),
    ("gpmppi_planner_create", C.c_int, [C.POINTER(MppiConfigC), C.POINTER(PredictionModelC),
                                        C.POINTER(NominalC), C.c_double, C.c_int, C.POINTER(_vp)]),
    ("gpmppi_planner_create_batch", C.c_int, [C.POINTER(MppiConfigC), C.POINTER(PredictionModelC),
                                              C.POINTER(NominalC), C.c_double, C.c_int,
                                              C.POINTER(C.c_uint64), C.c_int, C.POINTER(_vp)]),
    ("gpmppi_planner_free", None, [_vp]),
    ("gpmppi_planner_robots", C.c_int, [_vp]),
    ("gpmppi_planner_plan_step_batch", C.c_int, [_vp, _dp, C.POINTER(TaskC), _dp, C.POINTER(DiagC)]),
    ("gpmppi_planner_set_robot_terrain_weights", C.c_int, [_vp, C.c_int, _dp, C.c_int]),
    ("gpmppi_planner_plan_step", C.c_int, [_vp, _dp, C.POINTER(TaskC), _dp, C.POINTER(DiagC)]),
    ("gpmppi_planner_set_terrain_weights", C.c_int, [_vp, _dp, C.c_int]),
    ("gpmppi_planner_terrain_weights", C.c_int, [_vp, _dp]),
    ("gpmppi_planner_nominal_sequence", C.c_int, [_vp, _dp]),
    ("gpmppi_planner_set_nominal_sequence", C.c_int, [_vp, _dp]),
    ("gpmppi_planner_horizon_covariances", C.c_int, [_vp, _dp]),
    ("gpmppi_planner_lane_radii", C.c_int, [_vp, _dp]),
    ("gpmppi_planner_obstacle_margins", C.c_int, [_vp, _dp]),
    ("gpmppi_planner_set_thresholds", C.c_int, [_vp, _dp, _dp, C.c_int]),
    ("gpmppi_planner_tick", C.c_uint64, [_vp]),
    ("gpmppi_planner_horizon", C.c_int, [_vp]),
    ("gpmppi_planner_samples", C.c_int, [_vp]),
    ("gpmppi_planner_set_noise_mode", C.c_int, [_vp, C.c_int]),
    ("gpmppi_planner_inject_noise", C.c_int, [_vp, _dp]),
    ("gpmppi_planner_philox_noise", C.c_int, [_vp, C.c_uint64, _dp]),
    ("gpmppi_planner_sample_costs", C.c_int, [_vp, _dp]),
    ("gpmppi_planner_sample_weights", C.c_int, [_vp, _dp]),
    ("gpmppi_planner_flags", C.c_int, [_vp, _u8p, _u8p, _u8p, _u8p]),
    ("gpmppi_planner_set_variance_path", C.c_int, [_vp, C.c_int]),
    ("gpmppi_planner_variance_path", C.c_int, [_vp]),
    ("gpmppi_planner_bench_device", C.c_int, [_vp, _dp, C.POINTER(TaskC), C.c_int, C.c_int, _dp,
                                              _dp]),
    ("gpmppi_flush_l2", C.c_int, [C.c_int]),
    ("gpmppi_planner_io_bytes", C.c_int, [_vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    ("gpmppi_debug_tc_profile", C.c_int, [_dp]),
    ("gpmppi_debug_tc_trace", C.c_int, [_dp]),
    ("gpmppi_debug_timeline", C.c_int, [_dp]),
    ("gpmppi_tuple_doubles", C.c_int, [C.c_int]),
    ("gpmppi_planner_set_shard", C.c_int, [_vp, C.c_int64, C.c_int64]),
    ("gpmppi_planner_plan_partial", C.c_int, [_vp, _dp, C.POINTER(TaskC), _vp]),
    ("gpmppi_planner_plan_finish", C.c_int, [_vp, _vp, C.c_int, _dp, C.POINTER(DiagC)]),
    ("gpmppi_nccl_unique_id", C.c_int, [_vp]),
    ("gpmppi_planner_attach_comm", C.c_int, [_vp, _vp, C.c_int, C.c_int]),
    ("gpmppi_planner_shard", C.c_int, [_vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                       C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    ("gpmppi_planner_set_command_first", C.c_int, [_vp, C.c_int]),
    ("gpmppi_planner_wait_tightening", C.c_int, [_vp, C.POINTER(DiagC)]),
    ("gpmppi_combine_tuples_host", C.c_int, [_dp, C.c_int, C.c_int, C.c_double, _dp]),
    ("gpmppi_rollout", C.c_int, [C.POINTER(PredictionModelC), C.POINTER(NominalC), _dp, C.c_int, _dp, _dp,
                                 C.c_int, C.c_int, _dp, _dp]),
    ("gpmppi_sample_perturbations", C.c_int, [C.POINTER(MppiConfigC), C.c_uint64, C.c_int, _dp]),
    ("gpmppi_trajectory_weights", C.c_int, [_dp, C.c_int64, C.c_double, C.c_int, _dp]),
    ("gpmppi_update_controls", C.c_int, [_dp, C.c_int, _dp, _dp, C.c_int64, _dp, _dp, C.c_int, _dp]),
    ("gpmppi_shift_horizon", C.c_int, [_dp, C.c_int, C.c_int, _dp]),
    ("gpmppi_select_kernel_grid", C.c_int, [_dp, _dp, C.c_int64, C.c_int64, C.c_int, _dp, _dp]),
    ("gpmppi_wrap_angle", C.c_double, [C.c_double]),
    ("gpmppi_step_nominal", C.c_int, [_dp, _dp, C.POINTER(NominalC), _dp]),
    ("gpmppi_step_kinematic_unicycle", C.c_int, [_dp, _dp, C.c_double, _dp]),
    ("gpmppi_step_edd5", C.c_int, [_dp, _dp, C.POINTER(Edd5C), C.c_double, C.c_double, _dp]),
    ("gpmppi_jacobian_nominal", C.c_int, [_dp, _dp, C.POINTER(NominalC), _dp]),
    ("gpmppi_body_frame_displacement", C.c_int, [_dp, _dp, _dp]),
    ("gpmppi_kernel_eval", C.c_int, [_dp, _dp, _dp, _dp]),
    ("gpmppi_ensemble_combine", C.c_int, [_dp, _dp, _dp, C.c_int, _dp, _dp]),
    ("gpmppi_project_simplex", C.c_int, [_dp, C.c_int, _dp]),
    ("gpmppi_chi2_quantile_2dof", C.c_int, [C.c_double, _dp]),
    ("gpmppi_normal_quantile", C.c_int, [C.c_double, _dp]),
    ("gpmppi_normal_cdf", C.c_double, [C.c_double]),
    ("gpmppi_tighten_lane_radius", C.c_int, [C.c_double, _dp, C.c_double, _dp]),
    ("gpmppi_tighten_obstacle_distance", C.c_int, [_dp, _dp, C.c_double, _dp, C.c_double, _dp, _dp,
                                                   C.POINTER(C.c_int), _dp]),
]


def lib():
    """Load the in-tree library (raises if it was not built)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} missing: build it with `python -m paper_2411_03289_b200.build` "
                "(no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _LIB = L
    return _LIB


def check(rc: int) -> None:
    if rc == OK:
        return
    msg = lib().gpmppi_last_error().decode()
    if rc == INVALID_ARGUMENT:
        raise ValueError(msg)
    if rc == CUDA_ERROR:
        raise CudaError(msg)
    raise RuntimeError(msg)


def dptr(a):
    return None if a is None else a.ctypes.data_as(_dp)


def u8ptr(a):
    return None if a is None else a.ctypes.data_as(_u8p)
