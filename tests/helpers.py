"""Shared builders for parity tests: the same workload on the oracle and on the device."""
from __future__ import annotations

import numpy as np

from oracle import oracle as O
from paper_2411_03289_b200 import workloads as W

# Parity tolerances (stated):
#  - GP-mean / dynamics / tightening are FP64 on both sides → 1e-9 relative.
#  - the per-sample variance term comes from the FP32 variance kernel: its cost
#    contribution is α0·Σ_k trace ≤ ~1e-2 with relative error ≤ ~1e-4, so the
#    cost tolerance is atol 1e-6 + rtol 1e-9.
COST_ATOL, COST_RTOL = 1e-6, 1e-9
SEQ_ATOL = 1e-6          # nominal sequence / command (softmax amplifies cost error by 1/λ)
TIGHT_RTOL = 1e-7        # r̄, margins, horizon covariances


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


def assert_tick_parity(po, pd, flags_exact=True, label=""):
    co, cd = po.costs(), pd.sample_costs()
    fin_o, fin_d = np.isfinite(co), np.isfinite(cd)
    assert np.array_equal(fin_o, fin_d), f"{label}: finite masks differ"
    np.testing.assert_allclose(cd[fin_d], co[fin_o], rtol=COST_RTOL, atol=COST_ATOL,
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
    np.testing.assert_allclose(pd.nominal_sequence(), po.nominal_sequence(), atol=SEQ_ATOL,
                               rtol=0, err_msg=f"{label}: nominal sequence")
