"""Shared builders for parity tests: the same workload on the oracle and on the device."""
from __future__ import annotations

import numpy as np

from oracle import oracle as O
from paper_2411_03289_b200 import workloads as W

# Parity tolerances (stated):
#  - GP mean / dynamics / tightening are FP64 on both sides (agree to ~1e-12).
#  - the per-sample variance term comes from the tensor-core variance kernel (default
#    3xFP16; 3xTF32 and FFMA selectable). Its per-step error is bounded relative to the
#    signal variance: |Δvar| <= VAR_REL * sf2 (measured 2.0e-5 * sf2 for 3xFP16 at n=2048,
#    tests/test_gpu_variance_paths.py). The cost adds α0 · Σ_k Σ_g (Σ_o w_o²) var_g, so a
#    cost differs by at most α0 · T · sf2 · VAR_REL (Σ w² <= 1 on the simplex):
#    cost_atol(w) = COST_ATOL + α0·T·sf2·VAR_REL; at the test kernel (sf2 = 4e-3, T = 40,
#    α0 = 0.1) that is 1e-6 + 8e-9.
COST_ATOL, COST_RTOL = 1e-6, 1e-9
VAR_REL = 5e-5
SEQ_ATOL = 1e-6          # nominal sequence / command (softmax amplifies cost error by 1/λ)
TIGHT_RTOL = 1e-7        # r̄, margins, horizon covariances
# diagnostics: best / mean cost carry the cost tolerance; ESS and entropy are sums of the
# softmax weights, whose relative error is |Δc|/λ <= 1e-5 at λ = 0.1 (same bound as the
# weights, which are checked at rtol 1e-4)
DIAG_RTOL = 1e-5


def cost_atol(alpha0=0.1, T=40, sf2=4e-3):
    return COST_ATOL + alpha0 * T * sf2 * VAR_REL


def assert_diag_parity(do_, dd, label="", cost_tol=COST_ATOL):
    """StepDiagnostics of one tick (mppi.cpp:435-459) against the oracle's."""
    assert dd.nonfinite_samples == do_["nonfinite_samples"], f"{label}: nonfinite count"
    assert bool(dd.tightening_infeasible) == bool(do_["tightening_infeasible"]), f"{label}: infeasible"
    for k in ("best_cost", "mean_cost"):
        a, b = getattr(dd, k), do_[k]
        if np.isfinite(b):
            assert abs(a - b) <= cost_tol + COST_RTOL * abs(b), f"{label}: {k} {a} vs {b}"
        else:
            assert (np.isnan(a) and np.isnan(b)) or a == b, f"{label}: {k} {a} vs {b}"
    rtol = DIAG_RTOL * max(1.0, cost_tol / COST_ATOL)  # weight error scales with the cost error
    for k in ("ess", "weight_entropy"):
        a, b = getattr(dd, k), do_[k]
        assert abs(a - b) <= rtol * abs(b) + 1e-12, f"{label}: {k} {a} vs {b}"
    assert dd.command_ms > 0.0 and dd.plan_ms >= dd.command_ms, f"{label}: timings"


def oracle_task(w, obstacles):
    kind = {"tracking": O.ORC_TASK_TRACKING, "avoidance": O.ORC_TASK_AVOIDANCE,
            "combined": O.ORC_TASK_COMBINED}[w.task]
    if w.track == "circle":
        track = O.make_track("circle", (0.0, 0.0), 2.0, 0.4)
    else:
        track = O.make_track("poly", half_width=0.4, waypoints=[[0.0, 0.0], [60.0, 0.0]],
                             closed=False)
    return O.make_task(kind, track if w.task != "avoidance" else None, w.v_desired,
                       obstacles=obstacles if len(obstacles) else None, goal=(8.0, 0.0, 0.5))


def build_pair(w, gp_seed=0, samples=None, threads=0, var_path=None):
    """Returns (oracle_planner, device_planner, oracle_task, device_task, gp_data)."""
    import paper_2411_03289_b200 as G
    K = samples or w.samples
    task_d, _, obstacles = W.make_task_objects(w, G)
    task_o = oracle_task(w, obstacles)
    cfg = G.MppiConfig(samples=K, horizon=w.horizon, lam=w.lam, sigma_sim=w.sigma_sim,
                       seed=w.seed)
    data = None
    if w.model == "gp":
        X, Y, Kp = W.gp_training_set(w.n_points, w.terrains, seed=gp_seed)
        gp_o = O.GP(X, Y, Kp)
        gp_d = G.GpModel.fit(X, Y, Kp)
        data = (X, Y, Kp, gp_o, gp_d)
        po = O.Planner(K, w.horizon, O.ORC_MODEL_GP, gp_o, w.terrains, lam=w.lam,
                       sigma_sim=w.sigma_sim, seed=w.seed, threads=threads, p_x=w.p_x)
        pd = G.Planner(cfg, G.GpEnsemble(gp_d, w.terrains), p_x=w.p_x)
        if var_path is not None:
            pd.set_variance_path(var_path)
    else:
        kind_o = {"nominal": O.ORC_MODEL_NOMINAL, "unicycle": O.ORC_MODEL_UNICYCLE,
                  "edd5": O.ORC_MODEL_EDD5}[w.model]
        edd = (0.9, 0.95, 0.02, -0.2, 0.21)
        po = O.Planner(K, w.horizon, kind_o, None, 0, lam=w.lam, sigma_sim=w.sigma_sim,
                       seed=w.seed, threads=threads, p_x=w.p_x, edd5=edd, track_width=0.4)
        model = {"nominal": G.NominalDynamic(), "unicycle": G.UnicycleBaseline(),
                 "edd5": G.Edd5Baseline(G.Edd5Params(*edd), 0.4)}[w.model]
        pd = G.Planner(cfg, model, p_x=w.p_x)
    return po, pd, task_o, task_d, data


def assert_tick_parity(po, pd, flags_exact=True, label="", cost_tol=None, seq_tol=None):
    co, cd = po.costs(), pd.sample_costs()
    fin_o, fin_d = np.isfinite(co), np.isfinite(cd)
    assert np.array_equal(fin_o, fin_d), f"{label}: finite masks differ"
    np.testing.assert_allclose(cd[fin_d], co[fin_o], rtol=COST_RTOL, atol=cost_tol or COST_ATOL,
                               err_msg=f"{label}: per-sample costs")
    if fin_o.any():
        assert int(np.nanargmin(co)) == int(np.nanargmin(cd)), f"{label}: argmin sample"
    fo, fd = po.flags(), pd.flags()
    assert np.array_equal(fo["alive"], fd["alive"]), f"{label}: alive flags"
    assert np.array_equal(fo["terminal"], fd["terminal"]), f"{label}: terminal flags"
    if flags_exact:
        assert np.array_equal(fo["viol"], fd["viol"]), f"{label}: lane-violation flags"
        assert np.array_equal(fo["coll"], fd["coll"]), f"{label}: collision flags"
    wo, wd = po.weights(), pd.sample_weights()
    np.testing.assert_allclose(wd, wo, rtol=1e-4, atol=1e-9, err_msg=f"{label}: weights")
    np.testing.assert_allclose(pd.nominal_sequence(), po.nominal_sequence(), atol=seq_tol or SEQ_ATOL,
                               rtol=0, err_msg=f"{label}: nominal sequence")
