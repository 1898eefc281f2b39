"""B200-native GP-MPPI solve path (arXiv 2411.03289), drop-in for the reference
planner's plan_step. Host API mirrors /root/reference/proj/include/gpmppi/*.hpp;
compute runs in lib/libgpmppi_b200.so (sm_100a CUDA) through a C ABI."""
from .gpmppi import (  # noqa: F401
    AvoidanceTask, AvoidanceWeights, CircleObstacle, CombinedTask, ControlBounds, Edd5Baseline,
    Edd5Params, GoalSpec, GpEnsemble, GpModel, KernelParams, MppiConfig, NominalDynamic,
    NominalParams, Planner, BatchPlanner, StepDiagnostics, Track, TrackingTask, TrackingWeights,
    UnicycleBaseline, apply_tuple, chi2_quantile_2dof, combine_tuples, flush_l2,
    kernel_launches, nccl_unique_id, shard_range, tuple_doubles, RolloutResult, rollout, sample_perturbations,
    trajectory_weights, update_controls, shift_horizon, TrainedModels, load_models, save_models)
from ._capi import (  # noqa: F401
    NOISE_INJECTED, NOISE_PHILOX, VAR_FFMA, VAR_TC_1XTF32, VAR_TC_3XF16, VAR_TC_3XF16_PAIR, VAR_TC_3XTF32,
    CudaError)

from .harness import (  # noqa: F401
    ExperimentConfig, HistoryBuffer, RunMetrics, Scenario, TerrainProfile, WeightSolverConfig,
    make_scenario, per_terrain_mean_prediction, project_simplex, run_avoidance,
    run_avoidance_experiment, run_tracking, run_tracking_experiment, solve_weights, train_models)

__version__ = "0.1.0"
