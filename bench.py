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
  e2e    = the same metric through the public plan_step with host buffers (H2D of
           x0 + task, D2H of command + diagnostics inside the timed span), closed loop
           (x <- step_nominal(x, u)) over max(K, 200) ticks, L2 flushed
           between ticks; full plan_step (reference semantics, tightening included) and,
           beside it, the time to command in command-first mode.
  N > 1  = BASELINE config 5: one solve of K_total = 1,048,576 samples (T=40, n=512)
           sharded over the N ranks (strong scaling), one ncclAllGather of the
           (2T+6)-double reduction tuples inside the library per tick. `--gpus N`
           without torchrun spawns the N ranks itself.
--impl reference: the reference algorithm's FP64 CPU restatement (oracle/; the
           reference itself needs Eigen and cannot be built here) built -march=native
           on the host that runs it, OpenBLAS GEMM/TRMM standing in for Eigen's,
           all host threads, 128-sample chunks as mppi.cpp:401-426, same workload
           (a bounded sample of K when one CPU tick would take seconds).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# one metric string for both arms (the driver divides the two lines' values)
METRIC = "GP-MPPI solve throughput, sample-rollout-steps/s (p50/p99 solve latency ms in p50_ms/p99_ms)"
UNIT = "sample-rollout-steps/s"
SHARDED_K = 1 << 20  # config 5 at N > 1: north star "K >= 1M"
E2E_MIN_TICKS = 200  # >= 200 closed-loop ticks for p50/p99
CPU_SAMPLE_MAX_K = 16384  # bounded CPU sample per tick (the metric is a rate)


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


def load_fp64_peak(peaks):
    """Measured FP64 FMA throughput (tools/micro/fp64_peak.cu on a B200, committed under
    profiles/), else the spec figure 148 SM x 64 DFMA/clk x 2 x max clock."""
    try:
        with open(os.path.join(ROOT, "profiles", "fp64_peak.json")) as f:
            d = json.load(f)
        return float(d["fp64_fma_tflops"]), "measured DFMA (profiles/fp64_peak.json, tools/micro/fp64_peak.cu)"
    except Exception:
        return 148 * 64 * 2 * peaks.get("sm_max_mhz", 1965.0) * 1e6 / 1e12, \
            "spec: 148 SM x 64 DFMA x 2 x max clock (no measured DFMA peak found)"


def roofline_block(w, phase, steps, peaks, peaks_kind, var_path=3):
    """Roofline of the dominant kernel (SURVEY §8(d) algorithmic work per unit).

    unit = one sample-rollout-step; F = n² + 24n FLOP split as
      variance kernel: n(n+1) (triangular ||L^-1 k*||²) + 2n (squares, sum)
      rollout kernel:  22n (kernel-row dot 4n FMA + exponent offsets, mean 6n FMA) + n exp
    The rollout is FP64 (bound "fp64", against the measured DFMA peak); the variance is
    tensor-core work (bound "tensor", against the measured bf16 = fp16 dense peak).
    `frac_bf16` states every kernel against the contract's bf16 denominator as well.
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
    bf16 = peaks.get("bf16_tflops", 1590.0)
    fp64, fp64_kind = load_fp64_peak(peaks)
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            traffic_tab = json.load(f).get(w.name, {})
    except Exception:
        traffic_tab = {}
    tick_ms = sum(phase) / steps
    # 3xFP16 / 3xTF32 issue three tensor products per algorithmic MAC; FP16 runs at the bf16
    # dense rate, TF32 at half of it
    if var_path in (3, 4):
        # the CTA-pair kernel (tcgen05 cta_group::2) is path 4, and path 3's choice at n_pad > 256
        # (kernels_tc.cu launch_tc_variance)
        n_pad = (n + 15) // 16 * 16
        pair = var_path == 4 or n_pad > 256
        var = {"kernel": "variance_f16x2_kernel" if pair else "variance_f16_kernel", "bound": "tensor",
               "peak": bf16, "unit": "TFLOP/s",
               "peak_kind": f"{peaks_kind} fp16 dense = bf16 dense burst (MEASURED_PEAKS.json)"}
    elif var_path in (1, 2):
        var = {"kernel": "variance_tc2u_kernel", "bound": "tensor", "peak": bf16 / 2, "unit": "TFLOP/s",
               "peak_kind": f"tf32 dense = {peaks_kind} bf16 dense / 2"}
    else:
        var = {"kernel": "variance_ffma_kernel", "bound": "fp32", "unit": "TFLOP/s",
               "peak": 148 * 128 * 2 * peaks.get("sm_max_mhz", 1965.0) * 1e6 / 1e12,
               "peak_kind": "fp32 spec (148 SM x 128 FFMA x 2 x max clock)"}
    var.update({"launch_ms": var_ms, "flop_per_launch": units * (n * n + 3 * n),
                "tensor_issue_factor": 3 if var_path in (1, 3, 4) else 1})
    roll = {"kernel": "rollout_gp_kernel", "bound": "fp64", "peak": fp64, "unit": "TFLOP/s",
            "peak_kind": fp64_kind, "launch_ms": roll_ms, "flop_per_launch": units * 22 * n,
            "binding_resource": "FP64 pipe + shared-memory wavefronts + issue (ncu at config2, "
                                "profiles/r02/r2f: FP64 48%, LSU shared 58%, issue 51%; 7 warps/SM, "
                                "latency-bound)"}
    for k in (var, roll):
        k["achieved"] = k["flop_per_launch"] / (k["launch_ms"] / 1e3) / 1e12
        k["frac"] = k["achieved"] / k["peak"]
        k["frac_bf16"] = k["achieved"] / bf16
        k["phase_share"] = k["launch_ms"] / tick_ms
        k["traffic"] = traffic_tab.get(k["kernel"])
    dom = var if var_ms >= roll_ms else roll
    out = {key: dom[key] for key in ("bound", "kernel", "achieved", "peak", "unit", "frac", "traffic")}
    out.update({"peak_kind": dom["peak_kind"], "flop_per_launch": dom["flop_per_launch"],
                "launch_ms": dom["launch_ms"], "frac_bf16": dom["frac_bf16"],
                "phase_share": dom["phase_share"],
                "kernels": {"rollout_gp_kernel": roll, var["kernel"]: var}})
    return out


def workload(args):
    """The bench's workload: --config (default config2 at N=1, config5 at N>1), --samples."""
    import dataclasses

    from paper_2411_03289_b200 import workloads as W
    name = args.config or ("config5" if args.gpus > 1 else "config2")
    w = W.CONFIGS[name]
    K = args.samples or (SHARDED_K if args.gpus > 1 and name == "config5" else w.samples)
    return dataclasses.replace(w, samples=K)


def build_planner(w, api, var_path=None):
    """(planner, task, x0); a BatchPlanner with per-robot tasks / states when w.robots > 1."""
    from paper_2411_03289_b200 import workloads as W
    cfg = api.MppiConfig(samples=w.samples, horizon=w.horizon, lam=w.lam,
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


def _cpu_oracle():
    """The timed CPU path: oracle built -march=native here (falls back to the portable
    build if gcc is missing), with OpenBLAS GEMM/TRMM. Returns (module, description)."""
    native = subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "native"],
                            capture_output=True).returncode == 0
    os.environ["GPMPPI_ORACLE_NATIVE"] = "1" if native else "0"
    from oracle import oracle as O
    blas = O.use_blas(True)
    return O, f"{'-march=native' if native else '-march=x86-64-v3'} build, {blas}"


def cpu_reference(w, steps, warmup, threads=0, samples=None):
    """The reference algorithm's CPU restatement, timed on this host's cores."""
    O, how = _cpu_oracle()
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
    return ms, p.threads_used(), K, how


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown CPU"


def run_reference_arm(args, w):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    K = min(w.samples, CPU_SAMPLE_MAX_K)
    steps = args.steps if K == w.samples else max(3, min(args.steps, 5))
    ms, threads, K, how = cpu_reference(w, steps, 1, 0, samples=K)
    mean_ms = statistics.mean(ms)
    value = K * w.horizon / (mean_ms / 1e3)
    sample = (f"{steps} full plan_step ticks of {w.name} at K={K}"
              + (f" (bounded sample of K={w.samples}; the metric is a rate)" if K != w.samples else "")
              + (f", one robot of {w.robots}" if w.robots > 1 else "")
              + f" on {threads} threads; {how}; {_cpu_model()}")
    line = {
        "impl": "reference", "metric": METRIC,
        "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": steps,
        "warmup": args.warmup, "ms_per_step": mean_ms, "p50_ms": _percentile(ms, 50),
        "p99_ms": _percentile(ms, 99), "higher_is_better": True,
        "scaling": "strong" if args.gpus > 1 else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{w.name}: K={w.samples} T={w.horizon} M={w.n_points} R={w.terrains} "
                   f"task={w.task} obstacles={w.n_obstacles}", "samples": w.samples, "horizon": w.horizon,
                   "gp_points": w.n_points, "timed_samples": K},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


class _DryPlanner:
    def variance_path(self):
        return 3


class _DryClock:
    def summary(self):
        return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["dry run"]}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def spawn_ranks(args):
    """`--gpus N` without torchrun: launch the N ranks (one per GPU) ourselves."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)]
    cmd += sys.argv[1:]
    return subprocess.run(cmd).returncode


def _device_mem_used_gb():
    """Device memory in use (whole GPU, cudaMemGetInfo) after the planner is built and warm."""
    try:
        import torch
        free, total = torch.cuda.mem_get_info(0)
        return (total - free) / 1e9
    except Exception:
        return None


def e2e_loop(planner, task, x0, ticks, api, nominal, command_first=False):
    """Closed loop through the public plan_step: x <- step_nominal(x, u) after each tick
    (acceptance.cpp:437-442), L2 flushed between ticks (outside the span)."""
    from paper_2411_03289_b200 import harness as H
    planner.set_command_first(command_first)
    x = np.array(x0, dtype=np.float64)
    wall, cmd_ms, plan_ms = [], [], []
    d = api.StepDiagnostics()
    for _ in range(ticks):
        api.flush_l2(0)
        t0 = time.perf_counter()
        u = planner.plan_step(x, task, d)
        wall.append((time.perf_counter() - t0) * 1e3)
        cmd_ms.append(d.command_ms)
        if command_first:
            planner.wait_tightening(d)
        plan_ms.append(d.plan_ms)
        x = np.array(H.step_nominal(tuple(x), (float(u[0]), float(u[1])), nominal))
        if not np.all(np.isfinite(x)):
            x = np.array(x0, dtype=np.float64)
    planner.set_command_first(False)
    return wall, cmd_ms, plan_ms


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=None, help="config1..config5 (default config2; config5 at N>1)")
    ap.add_argument("--samples", type=int, default=None, help="override K (samples per robot per solve)")
    ap.add_argument("--variance-path", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-steps", type=int, default=3)
    ap.add_argument("--e2e-ticks", type=int, default=None)
    ap.add_argument("--sharded", action="store_true",
                    help="run the sharded (in-library NCCL) path even at one rank")
    ap.add_argument("--dry-run", action="store_true",
                    help="CPU contract check only: fake timings, no GPU, never a result")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    w = workload(args)
    if args.impl == "reference":
        run_reference_arm(args, w)
        return

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.gpus > 1 and world == 1 and not args.dry_run:
        sys.exit(spawn_ranks(args))
    if world > 1 or args.sharded or (args.dry_run and args.gpus > 1):
        run_sharded(args, w, max(world, args.gpus if args.dry_run else world), rank)
        return

    e2e_ticks = args.e2e_ticks or max(args.steps, E2E_MIN_TICKS)
    if args.dry_run:
        planner, clk = _DryPlanner(), _DryClock()
        tick_ms, phase = np.full(args.steps, 1.0), np.array([0.4, 0.35, 0.05, 0.2]) * args.steps
        launches = 7 * args.steps
        e2e_wall, e2e_cmd, e2e_plan = [1.1] * e2e_ticks, [0.9] * e2e_ticks, [1.0] * e2e_ticks
        cf_wall = [0.95] * e2e_ticks
        h2d, d2h = 2792, 132
        mem_gb = None
    else:
        import paper_2411_03289_b200 as G
        planner, task, x0 = build_planner(w, G, var_path=args.variance_path)
        for _ in range(args.warmup):
            planner.plan_step(x0, task)
        mem_gb = _device_mem_used_gb()
        launches0 = G.kernel_launches()
        with ClockSampler(0) as clk:
            tick_ms, phase = planner.bench_device(x0, task, args.steps, flush_l2=True)
        launches = G.kernel_launches() - launches0
        if w.robots > 1:  # batched planner: the public batched call, fixed states
            e2e_wall, e2e_cmd, e2e_plan = [], [], []
            diags = [G.StepDiagnostics() for _ in range(w.robots)]
            for _ in range(min(e2e_ticks, 20)):
                G.flush_l2(0)
                t0 = time.perf_counter()
                planner.plan_step(x0, task, diags)
                e2e_wall.append((time.perf_counter() - t0) * 1e3)
                e2e_cmd.append(diags[0].command_ms)
                e2e_plan.append(diags[0].plan_ms)
            cf_wall = None
        else:
            nominal = G.NominalParams()
            e2e_wall, e2e_cmd, e2e_plan = e2e_loop(planner, task, x0, e2e_ticks, G, nominal)
            cf_wall, _, _ = e2e_loop(planner, task, x0, e2e_ticks, G, nominal, command_first=True)
        h2d, d2h = planner.io_bytes()
    steps_per_tick = w.sample_steps  # robots x samples x horizon
    mean_ms = float(np.mean(tick_ms))
    value = steps_per_tick / (mean_ms / 1e3)
    e2e_value = steps_per_tick / (float(np.mean(e2e_wall)) / 1e3)
    peaks, peaks_kind = load_peaks()
    roofline = roofline_block(w, phase, args.steps, peaks, peaks_kind, planner.variance_path())
    n = w.n_points
    robots = f"{w.robots} robots x " if w.robots > 1 else ""
    e2e = {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
           "ticks": len(e2e_wall), "p50_ms": _percentile(e2e_wall, 50), "p99_ms": _percentile(e2e_wall, 99),
           "protocol": "closed loop x <- step_nominal(x, u), public plan_step with host buffers, "
                       "L2 flushed between ticks; full plan_step incl. tightening (reference plan_ms)",
           "plan_ms_p50": _percentile(e2e_plan, 50), "command_ms_p50": _percentile(e2e_cmd, 50),
           "command_ms_p99": _percentile(e2e_cmd, 99)}
    if cf_wall:
        e2e["command_first"] = {"p50_ms": _percentile(cf_wall, 50), "p99_ms": _percentile(cf_wall, 99),
                                "value": steps_per_tick / (float(np.mean(cf_wall)) / 1e3),
                                "note": "time to command: plan_step returns at the command, the "
                                        "tightening (next tick's input) completes behind it"}
    line = {
        "metric": METRIC,
        "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": mean_ms, "p50_ms": _percentile(tick_ms, 50),
        "p99_ms": _percentile(tick_ms, 99), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64+f32", "data": "synthetic",
        "config": {"workload": f"{w.name}: {robots}GP-MPPI path following + {w.n_obstacles} tightened "
                   f"obstacles, K={w.samples} T={w.horizon} M={n} R={w.terrains} p_x={w.p_x}",
                   "robots": w.robots, "samples": w.samples, "horizon": w.horizon, "gp_points": n,
                   "parallelism": "single GPU", "l2": "flushed between ticks (2x L2 memset)",
                   "variance_path": planner.variance_path(), "device_mem_used_gb": mem_gb,
                   "philox_noise": os.environ.get("GPMPPI_NOISE_MAT", "auto")},
        "phase_ms": {"rollout": phase[0] / args.steps, "variance": phase[1] / args.steps,
                     "reduce_update": phase[2] / args.steps, "tightening": phase[3] / args.steps},
        "e2e": e2e,
        "roofline": roofline,
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    if args.dry_run:
        line["dry_run"] = True
    if not args.no_cpu_baseline and not args.dry_run:
        K = min(w.samples, CPU_SAMPLE_MAX_K)
        ms, threads, K, how = cpu_reference(w, args.cpu_steps, 1, 0, samples=K)
        cpu_val = K * w.horizon / (statistics.mean(ms) / 1e3)
        line["cpu_baseline"] = {"value": cpu_val, "unit": UNIT, "cores": threads, "kind": "port",
                                "p50_ms": _percentile(ms, 50),
                                "sample": f"{args.cpu_steps} plan_step ticks of {w.name} (K={K}), "
                                          f"FP64 oracle, {threads} threads; {how}"}
    print(json.dumps(line), flush=True)


def run_sharded(args, w, world, rank):
    """Config 5 sharded over the ranks: K_total samples per solve, each rank its contiguous
    global range, the tuple all-gather over NCCL inside the library (no host sync per tick).
    torch.distributed (gloo, CPU) only bootstraps: id broadcast, barrier, max over ranks."""
    if args.dry_run:  # contract check of the N-rank line (no GPU, no ranks spawned)
        if rank == 0:
            print(json.dumps({"metric": METRIC, "value": 1.0, "unit": UNIT, "n_gpus": world,
                              "steps": args.steps, "warmup": args.warmup, "scaling": "strong",
                              "dry_run": True, "config": {"workload": f"{w.name} sharded: K={w.samples}"}}),
                  flush=True)
        return
    import torch
    import torch.distributed as dist

    import paper_2411_03289_b200 as G
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    if "MASTER_ADDR" not in os.environ:  # --sharded at one rank without torchrun
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()), RANK="0", WORLD_SIZE="1")
    dist.init_process_group("gloo")
    planner, task, x0 = build_planner(w, G)
    uid = [G.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    planner.attach_comm(uid[0], world, rank)
    for _ in range(args.warmup):
        planner.plan_step(x0, task)
    dist.barrier()
    launches0 = G.kernel_launches()
    with ClockSampler(local) as clk:
        tick_ms, phase = planner.bench_device(x0, task, args.steps, flush_l2=True)
    launches = G.kernel_launches() - launches0
    e2e_ticks = args.e2e_ticks or max(args.steps, 50)
    dist.barrier()
    e2e_wall, e2e_cmd, e2e_plan = e2e_loop(planner, task, x0, e2e_ticks, G, G.NominalParams())
    t = torch.tensor(np.concatenate([tick_ms, e2e_wall]), dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)  # every tick: the slowest rank
    tick_ms, e2e_wall = t[:len(tick_ms)].numpy(), t[len(tick_ms):].numpy()
    if rank == 0:
        mean_ms = float(tick_ms.mean())
        value = w.sample_steps / (mean_ms / 1e3)
        h2d, d2h = planner.io_bytes()
        begin, count, _, _ = planner.shard()
        line = {
            "metric": METRIC,
            "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": mean_ms, "p50_ms": _percentile(tick_ms, 50),
            "p99_ms": _percentile(tick_ms, 99), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64+f32", "data": "synthetic",
            "config": {"workload": f"{w.name} sharded: K={w.samples} total ({count} on rank 0) "
                       f"T={w.horizon} M={w.n_points} R={w.terrains} obstacles={w.n_obstacles}",
                       "samples": w.samples, "horizon": w.horizon, "gp_points": w.n_points,
                       "parallelism": f"sample-sharded x{world}, in-library ncclAllGather of the tuple",
                       "l2": "flushed between ticks (2x L2 memset)"},
            "phase_ms": {"rollout": phase[0] / args.steps, "variance": phase[1] / args.steps,
                         "reduce_exchange_update": phase[2] / args.steps,
                         "tightening": phase[3] / args.steps},
            "e2e": {"value": w.sample_steps / (float(np.mean(e2e_wall)) / 1e3), "unit": UNIT,
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ticks": len(e2e_wall),
                    "p50_ms": _percentile(e2e_wall, 50), "p99_ms": _percentile(e2e_wall, 99)},
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
