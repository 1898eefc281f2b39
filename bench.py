#!/usr/bin/env python
"""GP-MPPI solve benchmark (BASELINE.json metric) — one JSON line on rank 0.

Workload (N=1): BASELINE config 2 — GP-MPPI chance-constrained path following
+ 10 tightened circular obstacles, K=4096, T=40, M(=n GP points)=512, 3 terrains,
p_x=0.95; synthetic lane/obstacles, random-init GP of that shape (no datasets).
A "step" = one full plan_step (noise → rollout → variance → softmax update →
shift → tightening pass).

  value  = sample-rollout-steps/s over the timed ticks, device-resident inputs,
           CUDA events on the planner stream, L2 flushed between ticks (outside
           the timed spans), max over ranks.
  e2e    = the same metric through the public C-ABI plan_step with host buffers
           (H2D of x0 + task, D2H of command + diagnostics inside the timed span).
  N > 1  = sharded solve, weak scaling: K = 4096·N samples per solve, each rank
           rolls out 4096 (global-index Philox noise), one all-gather of the
           (2T+6)-double reduction tuple over NCCL, every rank finishes identically.
--impl reference: the reference algorithm's FP64 CPU restatement (oracle/, the
           reference itself needs Eigen and cannot be built here), all host
           threads, 128-sample chunks as mppi.cpp:401-426, same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def _percentile(xs, q):
    return float(np.percentile(np.asarray(xs, dtype=np.float64), q))


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([s.strip() for s in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def roofline_block(w, phase, steps, peaks, peaks_kind, var_path=3):
    """Roofline of the dominant kernel (SURVEY §8(d) algorithmic work per unit).

    unit = one sample-rollout-step; F = n² + 24n FLOP split as
      variance kernel: n(n+1) (triangular ||L^-1 k*||²) + 2n (squares, sum)
      rollout kernel:  22n (kernel-row dot 4n FMA + exponent offsets, mean 6n FMA) + n exp
    The contract's denominator is the measured bf16 dense peak; the path's own
    ceilings (FP16 dense = bf16 for the default 3xFP16 variance, TF32 dense = bf16/2 for
    3xTF32, FP64 = 148·64 DFMA·2·clock) are reported beside it.
    """
    n = w.n_points
    units = w.sample_steps
    if n == 0:  # GP-free model (config 1): one wave of thread-per-sample rollouts
        ms = phase[0] / steps
        words = (w.horizon + 31) // 32
        byts = w.robots * w.samples * (8 + 2 + 8 * words)  # costs, alive/terminal, flag words
        achieved = byts / (ms / 1e3) / 1e9
        peak = peaks.get("hbm_gbs", 6650.0)
        return {"bound": "hbm", "kernel": "rollout_base_kernel", "achieved": achieved, "peak": peak,
                "unit": "GB/s", "frac": achieved / peak, "traffic": None,
                "peak_kind": f"{peaks_kind} HBM copy (MEASURED_PEAKS.json)", "bytes_per_launch": byts,
                "launch_ms": ms, "phase_share": ms / (sum(phase) / steps),
                "note": "latency-bound: K=1024 samples are one wave of 40 serial FP64 steps"}
    roll_ms, var_ms = phase[0] / steps, phase[1] / steps
    peak = peaks.get("bf16_tflops", 1590.0)
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            traffic_tab = json.load(f).get(w.name, {})
    except Exception:
        traffic_tab = {}
    tick_ms = sum(phase) / steps
    # 3xFP16 / 3xTF32 issue three tensor products per algorithmic MAC; FP16 runs at the bf16
    # dense rate, TF32 at half of it
    bf16 = peaks.get("bf16_tflops", 1590.0)
    if var_path == 3:
        var = {"kernel": "variance_f16_kernel", "own_peak": bf16, "own_peak_kind": "fp16_dense_tflops (= bf16 dense)"}
    elif var_path in (1, 2):
        var = {"kernel": "variance_tc2u_kernel", "own_peak": bf16 / 2, "own_peak_kind": "tf32_dense_tflops (bf16/2)"}
    else:
        var = {"kernel": "variance_ffma_kernel", "own_peak": 148 * 128 * 2 * peaks.get("sm_max_mhz", 1965.0) * 1e6 / 1e12,
               "own_peak_kind": "fp32_tflops (148 SM x 128 FFMA x 2 x max clock)"}
    var.update({"bound": "tensor" if var_path else "fp32", "launch_ms": var_ms, "flop_per_launch": units * (n * n + 3 * n),
                "tensor_issue_factor": 3 if var_path in (1, 3) else 1})
    roll = {"kernel": "rollout_gp_kernel", "bound": "tensor", "launch_ms": roll_ms, "flop_per_launch": units * 22 * n,
            "own_peak": 148 * 64 * 2 * peaks.get("sm_max_mhz", 1965.0) * 1e6 / 1e12,
            "own_peak_kind": "fp64_tflops (148 SM x 64 DFMA x 2 x max clock)",
            "binding_resource": "FP64 pipe + shared-memory wavefronts + issue (ncu at config2: FP64 51%, LSU shared 60%; "
                                "7 warps/SM, latency-bound; config5: FP64 60%)"}
    for k in (var, roll):
        k["achieved"] = k["flop_per_launch"] / (k["launch_ms"] / 1e3) / 1e12
        k["peak"] = peak
        k["unit"] = "TFLOP/s"
        k["frac"] = k["achieved"] / peak
        k["frac_of_own_peak"] = k["achieved"] / k["own_peak"]
        k["phase_share"] = k["launch_ms"] / tick_ms
        k["traffic"] = traffic_tab.get(k["kernel"])
    dom = var if var_ms >= roll_ms else roll
    out = {key: dom[key] for key in ("bound", "kernel", "achieved", "peak", "unit", "frac", "traffic")}
    out.update({"peak_kind": f"{peaks_kind} bf16 dense burst (MEASURED_PEAKS.json)",
                "flop_per_launch": dom["flop_per_launch"], "launch_ms": dom["launch_ms"],
                "own_peak": dom["own_peak"], "own_peak_kind": dom["own_peak_kind"],
                "frac_of_own_peak": dom["frac_of_own_peak"], "phase_share": dom["phase_share"],
                "kernels": {"rollout_gp_kernel": roll, var["kernel"]: var}})
    return out


def build_planner(w, api, samples=None, var_path=None):
    """(planner, task, x0); a BatchPlanner with per-robot tasks / states when w.robots > 1."""
    from paper_2411_03289_b200 import workloads as W
    cfg = api.MppiConfig(samples=samples or w.samples, horizon=w.horizon, lam=w.lam,
                         sigma_sim=w.sigma_sim, seed=w.seed)
    if w.model == "gp":
        X, Y, K = W.gp_training_set(w.n_points, w.terrains, seed=0)
        gp = api.GpModel.fit(X, Y, K)
        model = api.GpEnsemble(gp, w.terrains)
    else:
        model = api.NominalDynamic()
    if w.robots > 1:
        p = api.BatchPlanner(cfg, model, w.robots, p_x=w.p_x)
        task, x0 = W.make_batch_tasks(w, api)
    else:
        p = api.Planner(cfg, model, p_x=w.p_x)
        task = W.make_task_objects(w, api)[0]
        x0 = np.array(w.x0, dtype=np.float64)
    if var_path is not None:
        p.set_variance_path(var_path)
    return p, task, x0


def cpu_reference(w, steps, warmup, threads=0, samples=None):
    """Oracle port of the reference algorithm, timed on this host's cores."""
    from oracle import oracle as O
    from paper_2411_03289_b200 import workloads as W
    from tests.helpers import oracle_task
    K = samples or w.samples
    X, Y, Kp = W.gp_training_set(w.n_points, w.terrains, seed=0)
    gp = O.GP(X, Y, Kp) if w.model == "gp" else None
    obstacles = W.random_obstacle_field(w.n_obstacles, seed=3) if w.n_obstacles else np.zeros((0, 3))
    to = oracle_task(w, obstacles)
    kind = O.ORC_MODEL_GP if w.model == "gp" else O.ORC_MODEL_NOMINAL
    p = O.Planner(K, w.horizon, kind, gp, w.terrains if gp else 0, lam=w.lam,
                  sigma_sim=w.sigma_sim, seed=w.seed, threads=threads, p_x=w.p_x)
    x = np.array(w.x0, dtype=np.float64)
    for _ in range(warmup):
        p.plan_step(x, to)
    ms = []
    for _ in range(steps):
        _, d = p.plan_step(x, to)
        ms.append(d["plan_ms"])
    return ms, p.threads_used(), K


def run_reference_arm(args, w):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    # bounded sample: full K per step when a tick is ~1 s, otherwise scale K down
    ms, threads, K = cpu_reference(w, args.steps, max(1, min(args.warmup, 1)), 0)
    mean_ms = statistics.mean(ms)
    value = K * w.horizon / (mean_ms / 1e3)
    cpu = subprocess.run(["bash", "-c", "lscpu | grep 'Model name' | head -1"], capture_output=True,
                         text=True).stdout.strip()
    line = {
        "impl": "reference", "metric": "sample-rollout-steps/s (GP-MPPI solve, p50/p99 ms in extra keys)",
        "value": value, "unit": "sample-rollout-steps/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": mean_ms, "p50_ms": _percentile(ms, 50),
        "p99_ms": _percentile(ms, 99), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{w.name}: K={K} T={w.horizon} n={w.n_points} R={w.terrains} "
                   f"task={w.task} obstacles={w.n_obstacles}", "samples": K, "horizon": w.horizon,
                   "gp_points": w.n_points},
        "cpu_baseline": {"value": value, "unit": "sample-rollout-steps/s", "cores": threads,
                         "kind": "port", "sample": f"{args.steps} full plan_step ticks of {w.name} "
                         f"(K={K}{', one robot of ' + str(w.robots) if w.robots > 1 else ''}) "
                         f"on {threads} threads; {cpu}"},
        "e2e": {"value": value, "unit": "sample-rollout-steps/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


class _DryPlanner:
    def variance_path(self):
        return 1


class _DryClock:
    def summary(self):
        return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["dry run"]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="config2")
    ap.add_argument("--variance-path", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-steps", type=int, default=3)
    ap.add_argument("--dry-run", action="store_true",
                    help="CPU contract check only: fake timings, no GPU, never a result")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    from paper_2411_03289_b200 import workloads as W
    w = W.CONFIGS[args.config]
    if args.impl == "reference":
        run_reference_arm(args, w)
        return

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        run_sharded(args, w, world, rank)
        return

    if args.dry_run:
        planner, clk = _DryPlanner(), _DryClock()
        tick_ms, phase = np.full(args.steps, 1.0), np.array([0.4, 0.35, 0.05, 0.2]) * args.steps
        launches, e2e_ms, (h2d, d2h) = 7 * args.steps, [1.1] * args.steps, (2768, 68)
    else:
        import paper_2411_03289_b200 as G
        planner, task, x0 = build_planner(w, G, var_path=args.variance_path)
        for _ in range(args.warmup):
            planner.plan_step(x0, task)
        launches0 = G.kernel_launches()
        with ClockSampler(0) as clk:
            tick_ms, phase = planner.bench_device(x0, task, args.steps, flush_l2=True)
        launches = G.kernel_launches() - launches0
        # e2e through the public plan_step (host buffers), L2 flushed between ticks
        e2e_ms = []
        for _ in range(args.steps):
            G.flush_l2(0)
            t0 = time.perf_counter()
            planner.plan_step(x0, task)
            e2e_ms.append((time.perf_counter() - t0) * 1e3)
        h2d, d2h = planner.io_bytes()
    steps_per_tick = w.sample_steps  # robots x samples x horizon
    mean_ms = float(np.mean(tick_ms))
    value = steps_per_tick / (mean_ms / 1e3)
    e2e_value = steps_per_tick / (float(np.mean(e2e_ms)) / 1e3)
    peaks, peaks_kind = load_peaks()
    roofline = roofline_block(w, phase, args.steps, peaks, peaks_kind, planner.variance_path())
    n = w.n_points
    rollout_ms, var_ms = phase[0] / args.steps, phase[1] / args.steps
    robots = f"{w.robots} robots x " if w.robots > 1 else ""
    line = {
        "metric": "sample-rollout-steps/s (GP-MPPI solve; p50/p99 latency in p50_ms/p99_ms)",
        "value": value, "unit": "sample-rollout-steps/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": mean_ms, "p50_ms": _percentile(tick_ms, 50),
        "p99_ms": _percentile(tick_ms, 99), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64+f32", "data": "synthetic",
        "config": {"workload": f"{w.name}: {robots}GP-MPPI path following + {w.n_obstacles} tightened "
                   f"obstacles, K={w.samples} T={w.horizon} M={n} R={w.terrains} p_x={w.p_x}",
                   "robots": w.robots, "samples": w.samples, "horizon": w.horizon, "gp_points": n,
                   "parallelism": "single GPU", "l2": "flushed between ticks (2x L2 memset)",
                   "variance_path": planner.variance_path()},
        "phase_ms": {"rollout": rollout_ms, "variance": var_ms,
                     "reduce_update": phase[2] / args.steps, "tightening": phase[3] / args.steps},
        "e2e": {"value": e2e_value, "unit": "sample-rollout-steps/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "p50_ms": _percentile(e2e_ms, 50),
                "p99_ms": _percentile(e2e_ms, 99)},
        "roofline": roofline,
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    if args.dry_run:
        line["dry_run"] = True
    if not args.no_cpu_baseline:
        ms, threads, K = cpu_reference(w, args.cpu_steps, 1, 0)
        cpu_val = K * w.horizon / (statistics.mean(ms) / 1e3)
        line["cpu_baseline"] = {"value": cpu_val, "unit": "sample-rollout-steps/s", "cores": threads,
                                "kind": "port", "p50_ms": _percentile(ms, 50),
                                "sample": f"{args.cpu_steps} plan_step ticks of {w.name} (K={K}), "
                                          f"FP64 oracle, {threads} threads"}
    print(json.dumps(line), flush=True)


def run_sharded(args, w, world, rank):
    """Weak-scaled sharded solve: K = w.samples·N, one NCCL all-gather per tick."""
    import torch
    import torch.distributed as dist

    import paper_2411_03289_b200 as G
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    K_total = w.samples * world
    planner, task, x0 = build_planner(w, G, samples=K_total)
    planner.set_shard(rank * w.samples, w.samples)
    W_t = G.tuple_doubles(w.horizon)
    mine = torch.zeros(W_t, dtype=torch.float64, device="cuda")
    gathered = torch.zeros(world, W_t, dtype=torch.float64, device="cuda")

    def tick():
        planner.plan_partial(x0, task, mine.data_ptr())
        dist.all_gather_into_tensor(gathered, mine)
        torch.cuda.current_stream().synchronize()
        return planner.plan_finish(gathered.data_ptr(), world)

    for _ in range(args.warmup):
        tick()
    dist.barrier()
    torch.cuda.synchronize()
    launches0 = G.kernel_launches()
    ms = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            tick()
            b.record()
            b.synchronize()
            ms.append(a.elapsed_time(b))
    dist.barrier()
    torch.cuda.synchronize()
    t = torch.tensor(ms, dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = t.cpu().numpy()
    launches = G.kernel_launches() - launches0
    if rank == 0:
        mean_ms = float(ms.mean())
        value = K_total * w.horizon / (mean_ms / 1e3)
        h2d, d2h = planner.io_bytes()
        line = {
            "metric": "sample-rollout-steps/s (GP-MPPI solve; p50/p99 latency in p50_ms/p99_ms)",
            "value": value, "unit": "sample-rollout-steps/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": mean_ms, "p50_ms": _percentile(ms, 50),
            "p99_ms": _percentile(ms, 99), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64+f32", "data": "synthetic",
            "config": {"workload": f"{w.name} sharded: K={K_total} ({w.samples}/GPU) T={w.horizon} "
                       f"M={w.n_points}", "samples": K_total, "horizon": w.horizon,
                       "gp_points": w.n_points, "parallelism": f"sample-sharded x{world}, NCCL all-gather",
                       "l2": "working set L2-resident; not flushed in the sharded loop"},
            "e2e": {"value": value, "unit": "sample-rollout-steps/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
