"""Sharded solve on one device: three planners own contiguous global
sample ranges of one K-sample solve, reduce them to tuples in device memory
(plan_partial), and every shard combines the stacked tuples in rank order
(plan_finish). Noise is keyed by the global sample index, so the shards must
reproduce the unsharded planner: per-sample costs within the oracle parity
tolerance (the rollout layout follows the shard size, so GP-mean partial sums are
grouped differently), the command and the updated sequence (1e-9), and
bit-identical results on every shard. The cross-process all-gather is covered by
tests/test_multirank_gloo.py; this checks the device side of the same protocol."""
import numpy as np
import pytest

from paper_2411_03289_b200 import workloads as W
from tests.helpers import COST_ATOL, COST_RTOL

pytestmark = pytest.mark.gpu


def test_three_shards_reproduce_the_unsharded_solve():
    import torch

    import paper_2411_03289_b200 as G
    w = W.CONFIGS["config2"]
    K, T = 3000, 24
    X, Y, Kp = W.gp_training_set(256, 3, seed=9)
    gp = G.GpModel.fit(X, Y, Kp)
    task = W.make_task_objects(w, G)[0]
    cfg = G.MppiConfig(samples=K, horizon=T, seed=21)
    full = G.Planner(cfg, G.GpEnsemble(gp, 3), p_x=0.95)
    shards = []
    for r in range(3):
        p = G.Planner(cfg, G.GpEnsemble(gp, 3), p_x=0.95)
        b, n = G.shard_range(K, 3, r)
        p.set_shard(b, n)
        shards.append((p, b, n))
    W_t = G.tuple_doubles(T)
    tuples = torch.zeros(3, W_t, dtype=torch.float64, device="cuda")
    x = np.array(w.x0, dtype=np.float64)
    for tick in range(3):
        u_full = full.plan_step(x, task)
        c_full = full.sample_costs()
        for r, (p, b, n) in enumerate(shards):
            p.plan_partial(x, task, tuples[r].data_ptr())
            np.testing.assert_allclose(p.sample_costs(), c_full[b:b + n], rtol=COST_RTOL, atol=COST_ATOL)
        torch.cuda.synchronize()
        cmds = [p.plan_finish(tuples.data_ptr(), 3) for p, _, _ in shards]
        for r in range(1, 3):
            np.testing.assert_array_equal(cmds[r], cmds[0])
            np.testing.assert_array_equal(shards[r][0].nominal_sequence(), shards[0][0].nominal_sequence())
        np.testing.assert_allclose(cmds[0], u_full, rtol=1e-9, atol=1e-9)
        np.testing.assert_allclose(shards[0][0].nominal_sequence(), full.nominal_sequence(), rtol=1e-9, atol=1e-9)
        np.testing.assert_allclose(shards[0][0].lane_radii(), full.lane_radii(), rtol=1e-10, atol=1e-14)
        x = x + np.array([0.02, 0.0, 0.0, 0.05, 0.0])
