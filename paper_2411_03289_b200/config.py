"""The reference's JSON experiment configuration (config.hpp:85-110, config.cpp).

`default_config()` / `load_config(path)` / `dump_config(cfg)` work on the canonical JSON
tree the reference writes (dump_config, config.cpp:430-519): every section present,
keys sorted as nlohmann::json orders them. `load_config` rejects unknown keys with the
reference's path-qualified messages (Section::finish, config.cpp:40-46) and validates
like ExperimentConfig::validate (config.cpp:126-185). `to_experiment` turns the tree into
the closed-loop driver's inputs (harness.ExperimentConfig + make_scenario arguments).

Host-side configuration parsing: not on the per-tick path.
"""
from __future__ import annotations

import copy
import json
import math

from . import gpmppi as G

PLANNERS = ("gp", "edd5", "unicycle")


def planner_kind(s: str) -> str:  # config.cpp:23-28
    if s not in PLANNERS:
        raise ValueError(f"unknown planner '{s}' (expected gp, edd5 or unicycle)")
    return s


def _terrains():  # config.cpp:116-124
    rows = [("tile", 0.97, 0.97, 0.45, 0.32, 0.05, 0.010, 0.020),
            ("asphalt", 0.92, 0.90, 0.55, 0.40, 0.15, 0.015, 0.030),
            ("grass", 0.82, 0.80, 0.70, 0.50, 0.35, 0.020, 0.040)]
    keys = ("name", "gain_v", "gain_omega", "tau_v_true", "tau_omega_true", "curvature_slip_c",
            "noise_std_v", "noise_std_omega")
    return [dict(zip(keys, r)) for r in rows]


def default_config() -> dict:
    """The default ExperimentConfig as its canonical JSON tree (config.hpp defaults)."""
    return {
        "seed": 0, "threads": 0, "planner": "gp",
        "nominal": {"tau_v": 0.5, "tau_omega": 0.35, "dt": 0.05},
        "terrains": _terrains(),
        "training": {"n_points": 300, "hold_min": 5, "hold_max": 20},
        "gp": {"hyperparams": "grid"},
        "estimator": {"history": 20, "gamma": 0.1, "max_iters": 200, "tol": 1e-8},
        "uncertainty": {"p_x": 0.95},
        "costs": {"tracking": {"variance": 0.1, "deviation": 1.0, "slip": 0.3, "safety": 1.0, "speed": 0.2},
                  "avoidance": {"variance": 0.1, "obstacle": 1.0, "stage": 0.5, "terminal": 1.0},
                  "high_cost": 1e4},
        "mppi": {"samples": 1024, "horizon": 30, "lambda": 0.1, "sigma_v_std": 0.3, "sigma_omega_std": 0.5,
                 "v_min": -0.5, "v_max": 2.0, "omega_min": -2.0, "omega_max": 2.0},
        "robot": {"track_width": 0.37},
        "geometry": {"circle": {"center": [0.0, 0.0], "radius": 2.0, "half_width": 0.4},
                     "square": {"center": [0.0, 0.0], "side": 6.25, "half_width": 0.4},
                     "lane": {"from": [0.0, 0.0], "to": [60.0, 0.0], "half_width": 0.4}},
        "scenario": {"kind": "tracking", "track": "circle", "v_desired": 2.0, "start": None,
                     "goal": {"position": [8.0, 0.0], "capture_radius": 0.5},
                     "random_obstacles": {"count": 5, "x_min": 1.5, "x_max": 6.5, "y_min": -2.5,
                                          "y_max": 2.5, "radius_min": 0.25, "radius_max": 0.5,
                                          "min_gap": 0.5},
                     "schedule": [{"time": 0.0, "terrain": 0}],
                     "distance_budget": 100.0, "max_duration": 120.0},
        "bench": {"planners": ["gp", "edd5", "unicycle"], "tracks": ["circle"], "terrains": [0, 1, 2],
                  "tracking_seeds": 1, "avoidance_trials": 33},
    }


def dump_config(cfg: dict) -> str:
    """Canonical text (config.cpp:430-519: nlohmann dump(2), keys in std::map order)."""
    return json.dumps(cfg, indent=2, sort_keys=True) + "\n"


def default_config_json() -> str:  # module.cpp:182
    return dump_config(default_config())


def config_hash_hex(cfg: dict) -> str:  # config.cpp:521-531 (FNV-1a of the canonical dump)
    h = 0xCBF29CE484222325
    for c in dump_config(cfg).encode():
        h = ((h ^ c) * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"


class _Section:  # config.cpp:34-90 strict object view
    def __init__(self, j, path):
        if not isinstance(j, dict):
            raise ValueError(f"config: {path} must be an object")
        self.j, self.path, self.seen = j, path, set()

    def has(self, key):
        self.seen.add(key)
        return key in self.j

    def at(self, key):
        return self.j[key]

    def get(self, key, target: dict, kind=None):
        if not self.has(key):
            return
        v = self.j[key]
        if kind is float and isinstance(v, (int, float)) and not isinstance(v, bool):
            v = float(v)
        elif kind is int and not (isinstance(v, int) and not isinstance(v, bool)):
            raise ValueError(f"config: bad value at '{self.path}.{key}'")
        elif kind is str and not isinstance(v, str):
            raise ValueError(f"config: bad value at '{self.path}.{key}'")
        elif kind is float and not isinstance(v, float):
            raise ValueError(f"config: bad value at '{self.path}.{key}'")
        target[key] = v

    def get_vec2(self, key, target: dict):
        if not self.has(key):
            return
        v = self.j[key]
        if not isinstance(v, list) or len(v) != 2:
            raise ValueError(f"config: '{self.path}.{key}' must have 2 entries")
        target[key] = [float(v[0]), float(v[1])]

    def finish(self):
        for k in self.j:
            if k not in self.seen:
                raise ValueError(f"config: unknown key '{self.path}.{k}'")


def _floats(sec: _Section, target: dict, keys):
    for k in keys:
        sec.get(k, target, float)


def load_config(path: str) -> dict:
    """config.cpp:187-428: defaults overlaid by the file, unknown keys rejected."""
    try:
        with open(path) as f:
            text = f.read()
    except OSError:
        raise RuntimeError(f"config: cannot open {path}")
    try:
        j = json.loads(text)
    except json.JSONDecodeError as e:
        raise ValueError(f"config: parse error in {path}: {e}")
    cfg = default_config()
    root = _Section(j, "$")
    root.get("seed", cfg, int)
    root.get("threads", cfg, int)
    if root.has("planner"):
        cfg["planner"] = planner_kind(root.at("planner"))
    if root.has("nominal"):
        s = _Section(root.at("nominal"), "$.nominal")
        _floats(s, cfg["nominal"], ("tau_v", "tau_omega", "dt"))
        s.finish()
    if root.has("terrains"):
        arr = root.at("terrains")
        if not isinstance(arr, list) or not arr:
            raise ValueError("config: terrains must be a non-empty array")
        cfg["terrains"] = []
        for i, t in enumerate(arr):
            s = _Section(t, f"$.terrains[{i}]")
            d = {"name": "", "gain_v": 1.0, "gain_omega": 1.0, "tau_v_true": 0.5, "tau_omega_true": 0.35,
                 "curvature_slip_c": 0.0, "noise_std_v": 0.0, "noise_std_omega": 0.0}
            s.get("name", d, str)
            _floats(s, d, ("gain_v", "gain_omega", "tau_v_true", "tau_omega_true", "curvature_slip_c",
                           "noise_std_v", "noise_std_omega"))
            s.finish()
            cfg["terrains"].append(d)
    if root.has("training"):
        s = _Section(root.at("training"), "$.training")
        for k in ("n_points", "hold_min", "hold_max"):
            s.get(k, cfg["training"], int)
        s.finish()
    if root.has("gp"):
        s = _Section(root.at("gp"), "$.gp")
        mode = {"hyperparams": "grid"}
        s.get("hyperparams", mode, str)
        if mode["hyperparams"] == "grid":
            if s.has("signal_var") or s.has("lengthscales") or s.has("noise_var"):
                raise ValueError("config: fixed kernel values only allowed with hyperparams=fixed")
            cfg["gp"] = {"hyperparams": "grid"}
        elif mode["hyperparams"] == "fixed":
            g = {"hyperparams": "fixed", "signal_var": 1.0, "lengthscales": [1.0, 1.0, 1.0, 1.0],
                 "noise_var": 1e-4}
            _floats(s, g, ("signal_var", "noise_var"))
            if s.has("lengthscales"):
                ls = s.at("lengthscales")
                if not isinstance(ls, list) or len(ls) != 4:
                    raise ValueError("config: gp.lengthscales must have 4 entries")
                g["lengthscales"] = [float(v) for v in ls]
            cfg["gp"] = g
        else:
            raise ValueError("config: gp.hyperparams must be grid or fixed")
        s.finish()
    if root.has("estimator"):
        s = _Section(root.at("estimator"), "$.estimator")
        s.get("history", cfg["estimator"], int)
        s.get("max_iters", cfg["estimator"], int)
        _floats(s, cfg["estimator"], ("gamma", "tol"))
        s.finish()
    if root.has("uncertainty"):
        s = _Section(root.at("uncertainty"), "$.uncertainty")
        _floats(s, cfg["uncertainty"], ("p_x",))
        s.finish()
    if root.has("costs"):
        s = _Section(root.at("costs"), "$.costs")
        if s.has("tracking"):
            t = _Section(s.at("tracking"), "$.costs.tracking")
            _floats(t, cfg["costs"]["tracking"], ("variance", "deviation", "slip", "safety", "speed"))
            t.finish()
        if s.has("avoidance"):
            a = _Section(s.at("avoidance"), "$.costs.avoidance")
            _floats(a, cfg["costs"]["avoidance"], ("variance", "obstacle", "stage", "terminal"))
            a.finish()
        _floats(s, cfg["costs"], ("high_cost",))
        s.finish()
    if root.has("mppi"):
        s = _Section(root.at("mppi"), "$.mppi")
        s.get("samples", cfg["mppi"], int)
        s.get("horizon", cfg["mppi"], int)
        _floats(s, cfg["mppi"], ("lambda", "sigma_v_std", "sigma_omega_std", "v_min", "v_max", "omega_min",
                                 "omega_max"))
        s.finish()
    if root.has("robot"):
        s = _Section(root.at("robot"), "$.robot")
        _floats(s, cfg["robot"], ("track_width",))
        s.finish()
    if root.has("geometry"):
        s = _Section(root.at("geometry"), "$.geometry")
        for name, vecs, scal in (("circle", ("center",), ("radius", "half_width")),
                                 ("square", ("center",), ("side", "half_width")),
                                 ("lane", ("from", "to"), ("half_width",))):
            if s.has(name):
                c = _Section(s.at(name), f"$.geometry.{name}")
                for v in vecs:
                    c.get_vec2(v, cfg["geometry"][name])
                _floats(c, cfg["geometry"][name], scal)
                c.finish()
        s.finish()
    if root.has("scenario"):
        s = _Section(root.at("scenario"), "$.scenario")
        sc = cfg["scenario"]
        s.get("kind", sc, str)
        s.get("track", sc, str)
        _floats(s, sc, ("v_desired",))
        if s.has("start"):
            st = s.at("start")
            if st is None:
                sc["start"] = None
            else:
                if not isinstance(st, list) or len(st) != 3:
                    raise ValueError("config: scenario.start must be [x, y, theta] or null")
                sc["start"] = [float(v) for v in st]
        if s.has("goal"):
            g = _Section(s.at("goal"), "$.scenario.goal")
            g.get_vec2("position", sc["goal"])
            _floats(g, sc["goal"], ("capture_radius",))
            g.finish()
        if s.has("obstacles"):
            obs = []
            for o in s.at("obstacles"):
                if not isinstance(o, list) or len(o) != 3:
                    raise ValueError("config: each obstacle must be [x, y, radius]")
                obs.append([float(v) for v in o])
            sc.pop("random_obstacles", None)
            sc["obstacles"] = obs
        if s.has("random_obstacles"):
            sc.pop("obstacles", None)
            ro = copy.deepcopy(default_config()["scenario"]["random_obstacles"])
            r = _Section(s.at("random_obstacles"), "$.scenario.random_obstacles")
            r.get("count", ro, int)
            _floats(r, ro, ("x_min", "x_max", "y_min", "y_max", "radius_min", "radius_max", "min_gap"))
            r.finish()
            sc["random_obstacles"] = ro
        if s.has("schedule"):
            sched = []
            for i, e in enumerate(s.at("schedule")):
                es = _Section(e, f"$.scenario.schedule[{i}]")
                d = {"time": 0.0, "terrain": 0}
                _floats(es, d, ("time",))
                es.get("terrain", d, int)
                es.finish()
                sched.append(d)
            sc["schedule"] = sched
        _floats(s, sc, ("distance_budget", "max_duration"))
        s.finish()
    if root.has("bench"):
        s = _Section(root.at("bench"), "$.bench")
        b = cfg["bench"]
        if s.has("planners"):
            b["planners"] = [planner_kind(p) for p in s.at("planners")]
        if s.has("tracks"):
            b["tracks"] = list(s.at("tracks"))
        if s.has("terrains"):
            b["terrains"] = [int(t) for t in s.at("terrains")]
        s.get("tracking_seeds", b, int)
        s.get("avoidance_trials", b, int)
        s.finish()
    root.finish()
    validate(cfg)
    return cfg


def validate(cfg: dict) -> None:  # config.cpp:126-185
    n = cfg["nominal"]
    if not (n["tau_v"] > 0.0) or not (n["tau_omega"] > 0.0):
        raise ValueError("NominalParams: time constants must be positive")
    if not (n["dt"] > 0.0) or n["dt"] >= min(n["tau_v"], n["tau_omega"]):
        raise ValueError("NominalParams: require 0 < dt < min(tau_v, tau_omega)")
    if not cfg["terrains"]:
        raise ValueError("config: at least one terrain profile required")
    for t in cfg["terrains"]:
        if not (0.0 < t["gain_v"] <= 1.2) or not (0.0 < t["gain_omega"] <= 1.2):
            raise ValueError("TerrainProfile: gains must lie in (0, 1.2]")
        if not (t["tau_v_true"] > 0.0) or not (t["tau_omega_true"] > 0.0):
            raise ValueError("TerrainProfile: time constants must be positive")
        if t["noise_std_v"] < 0.0 or t["noise_std_omega"] < 0.0:
            raise ValueError("TerrainProfile: noise stds must be >= 0")
    tr = cfg["training"]
    if tr["n_points"] < 1 or tr["hold_min"] < 1 or tr["hold_max"] < tr["hold_min"]:
        raise ValueError("config: bad training section")
    if cfg["gp"]["hyperparams"] == "fixed":
        g = cfg["gp"]
        if not (g["signal_var"] > 0.0) or not (g["noise_var"] > 0.0) or not all(v > 0.0 for v in g["lengthscales"]):
            raise ValueError("KernelParams: all parameters must be strictly positive")
    e = cfg["estimator"]
    if e["history"] < 1 or e["gamma"] < 0.0 or not (e["tol"] > 0.0) or e["max_iters"] < 1:
        raise ValueError("config: bad estimator section")
    p_x = cfg["uncertainty"]["p_x"]
    if not (p_x > 0.5) or not (p_x < 1.0):
        raise ValueError("config: p_x must lie in (0.5, 1)")
    for k, v in list(cfg["costs"]["tracking"].items()) + list(cfg["costs"]["avoidance"].items()):
        if not (v >= 0.0) or not math.isfinite(v):
            raise ValueError("costs: weights must be finite and non-negative")
    if not (cfg["costs"]["high_cost"] > 0.0):
        raise ValueError("config: high_cost must be positive")
    m = cfg["mppi"]
    if m["samples"] < 1 or m["horizon"] < 1:
        raise ValueError("MppiConfig: samples and horizon must be >= 1")
    if not (m["lambda"] > 0.0):
        raise ValueError("MppiConfig: lambda must be positive")
    if not (m["sigma_v_std"] > 0.0) or not (m["sigma_omega_std"] > 0.0):
        raise ValueError("MppiConfig: sampling variances must be positive")
    if m["v_min"] >= m["v_max"] or m["omega_min"] >= m["omega_max"]:
        raise ValueError("MppiConfig: control bounds must be a nonempty box")
    if not (cfg["robot"]["track_width"] > 0.0):
        raise ValueError("config: track_width must be positive")
    sc = cfg["scenario"]
    if sc["kind"] not in ("tracking", "avoidance"):
        raise ValueError("config: scenario.kind must be tracking or avoidance")
    if sc["track"] not in ("circle", "square", "lane"):
        raise ValueError("config: scenario.track must be circle, square or lane")
    if not sc["schedule"]:
        raise ValueError("config: scenario.schedule must be non-empty")
    prev = -1.0
    for e in sc["schedule"]:
        if e["time"] <= prev:
            raise ValueError("config: schedule times must be strictly increasing")
        prev = e["time"]
        if e["terrain"] < 0 or e["terrain"] >= len(cfg["terrains"]):
            raise ValueError("config: schedule references a missing terrain index")
    for t in cfg["bench"]["terrains"]:
        if t < 0 or t >= len(cfg["terrains"]):
            raise ValueError("config: bench references a missing terrain index")
    for tr_name in cfg["bench"]["tracks"]:
        if tr_name not in ("circle", "square"):
            raise ValueError("config: bench tracks must be circle or square")
    if cfg["bench"]["tracking_seeds"] < 1 or cfg["bench"]["avoidance_trials"] < 1:
        raise ValueError("config: bench counts must be >= 1")


def to_experiment(cfg: dict):
    """(harness.ExperimentConfig, make_scenario keyword arguments) of a config tree.
    `threads` is accepted and irrelevant: the planner's work runs on the GPU."""
    from . import harness as H
    validate(cfg)
    m = cfg["mppi"]
    mc = G.MppiConfig(samples=m["samples"], horizon=m["horizon"], lam=m["lambda"],
                      sigma_sim=(m["sigma_v_std"] ** 2, m["sigma_omega_std"] ** 2),
                      bounds=G.ControlBounds((m["v_min"], m["omega_min"]), (m["v_max"], m["omega_max"])),
                      seed=0, threads=cfg["threads"])
    g = cfg["gp"]
    fixed = G.KernelParams(g.get("signal_var", 1.0), tuple(g.get("lengthscales", (1.0,) * 4)),
                           g.get("noise_var", 1e-4))
    e = cfg["estimator"]
    tw, aw = cfg["costs"]["tracking"], cfg["costs"]["avoidance"]
    ec = H.ExperimentConfig(
        seed=cfg["seed"], planner=cfg["planner"], nominal=G.NominalParams(**cfg["nominal"]),
        terrains=[H.TerrainProfile(**t) for t in cfg["terrains"]],
        n_points=cfg["training"]["n_points"], hold_min=cfg["training"]["hold_min"],
        hold_max=cfg["training"]["hold_max"], grid_search=g["hyperparams"] == "grid", fixed_kernel=fixed,
        history=e["history"], gamma=e["gamma"], max_iters=e["max_iters"], tol=e["tol"],
        p_x=cfg["uncertainty"]["p_x"], tracking=G.TrackingWeights(**tw), avoidance=G.AvoidanceWeights(**aw),
        high_cost=cfg["costs"]["high_cost"], mppi=mc, track_width=cfg["robot"]["track_width"])
    sc = cfg["scenario"]
    kw = {"kind": sc["kind"], "track": sc["track"], "v_desired": sc["v_desired"],
          "schedule": [(float(x["time"]), int(x["terrain"])) for x in sc["schedule"]],
          "distance_budget": sc["distance_budget"], "max_duration": sc["max_duration"],
          "goal": G.GoalSpec(tuple(sc["goal"]["position"]), sc["goal"]["capture_radius"]),
          "geometry": cfg["geometry"], "start": sc["start"],
          "obstacles": sc.get("obstacles"), "random_obstacles": sc.get("random_obstacles")}
    return ec, kw
