"""Acceptance-style closed-loop runs on the device planner (acceptance.cpp:335-420 shape).

Criterion 7: tracking on the circle, 100 m budget, per terrain, gp vs edd5 vs unicycle
(gp must have the lowest RMSE; on grass < 0.6x unicycle). Criterion 8 (short): avoidance
success counts over a few seeded obstacle fields. Prints one JSON line per run.

  python tools/closed_loop.py [--budget 100] [--trials 5]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2411_03289_b200 import harness as H  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--budget", type=float, default=100.0)
    ap.add_argument("--trials", type=int, default=5)
    ap.add_argument("--samples", type=int, default=1024)
    ap.add_argument("--horizon", type=int, default=30)
    a = ap.parse_args()
    cfg = H.ExperimentConfig()
    cfg.mppi.samples, cfg.mppi.horizon = a.samples, a.horizon
    models = H.train_models(cfg, cfg.seed)
    for terrain in range(3):
        master = H.derive_seed(cfg.seed, 7000 + terrain)
        row = {"criterion": 7, "terrain": cfg.terrains[terrain].name}
        for kind in ("gp", "edd5", "unicycle"):
            c = H.ExperimentConfig(**{**cfg.__dict__, "planner": kind})
            sc = H.make_scenario("tracking", "circle", schedule=[(0.0, terrain)],
                                 distance_budget=a.budget, max_duration=180.0)
            m = H.run_tracking_experiment(c, sc, models, master)
            row[kind] = {"rmse": m.rmse, "success": m.success, "ticks": m.ticks,
                         "plan_ms_median": m.latency.median_ms, "aborted": m.abort_reason}
        row["gp_best"] = row["gp"]["rmse"] < min(row["edd5"]["rmse"], row["unicycle"]["rmse"])
        print(json.dumps(row), flush=True)
    for terrain in range(3):
        wins = {"gp": 0, "unicycle": 0}
        for trial in range(a.trials):
            seed = H.derive_seed(cfg.seed, 8000 + terrain, trial)
            sc = H.make_scenario("avoidance", seed=seed, schedule=[(0.0, terrain)])
            for kind in wins:
                c = H.ExperimentConfig(**{**cfg.__dict__, "planner": kind})
                wins[kind] += H.run_avoidance_experiment(c, sc, models, seed).success
        print(json.dumps({"criterion": 8, "terrain": cfg.terrains[terrain].name,
                          "trials": a.trials, "successes": wins}), flush=True)


if __name__ == "__main__":
    main()
