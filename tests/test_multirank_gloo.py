"""CPU multi-rank (world_size 2, gloo) test of the sharded solve's host logic
(SURVEY §8(e)): contiguous global shards, per-rank reduction tuples, one
all-gather, rank-order combine, update/clamp/shift — against the single-process
oracle update (mppi.cpp:125-173) on the same costs and noise."""
import os
import socket

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp

LAM, T, K = 0.1, 9, 301


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_tuple(c, e):
    f = np.isfinite(c)
    m = c[f].min() if f.any() else np.inf
    ex = np.zeros_like(c)
    ex[f] = np.exp(-(c[f] - m) / LAM)
    head = [m, ex.sum(), (ex * ex).sum(), (ex[f] * (c[f] - m)).sum(), float(f.sum()), c[f].sum()]
    return np.concatenate([head, (ex[:, None, None] * e).sum(0).ravel()])


def _worker(rank, world, port, out):
    import torch
    import paper_2411_03289_b200 as G
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(42)
    costs = rng.uniform(0, 3, K)
    costs[[5, 200]] = np.nan
    eps = 0.3 * rng.standard_normal((K, T, 2))
    nominal = rng.uniform(-0.5, 1.5, (T, 2))
    b, n = G.shard_range(K, world, rank)
    mine = torch.from_numpy(_rank_tuple(costs[b:b + n], eps[b:b + n]))
    gathered = [torch.zeros_like(mine) for _ in range(world)]
    dist.all_gather(gathered, mine)
    comb = G.combine_tuples(torch.stack(gathered).numpy(), T, LAM)
    cmd, seq = G.apply_tuple(comb, nominal)
    out[rank] = (cmd, seq, comb)
    dist.destroy_process_group()


def test_two_rank_sharded_update_matches_single_process_oracle():
    from oracle import oracle as O
    import paper_2411_03289_b200 as G
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    rng = np.random.default_rng(42)
    costs = rng.uniform(0, 3, K)
    costs[[5, 200]] = np.nan
    eps = 0.3 * rng.standard_normal((K, T, 2))
    nominal = rng.uniform(-0.5, 1.5, (T, 2))
    w = np.empty(K)
    O.lib().orc_trajectory_weights(O._ptr(costs), K, LAM, O._ptr(w))
    upd = np.empty((T, 2))
    e = np.ascontiguousarray(eps)
    O.lib().orc_update_controls(O._ptr(nominal), O._ptr(e), O._ptr(w), K, T, O._ptr(np.array([-0.5, -2.0])),
                                O._ptr(np.array([2.0, 2.0])), O._ptr(upd))
    shifted = np.empty((T, 2))
    O.lib().orc_shift_horizon(O._ptr(upd), T, O._ptr(shifted))
    for r in range(2):
        cmd, seq, comb = out[r]
        np.testing.assert_allclose(cmd, upd[0], rtol=0, atol=1e-13)
        np.testing.assert_allclose(seq, shifted, rtol=0, atol=1e-13)
        assert comb[4] == K - 2  # finite count
        ess = comb[1] ** 2 / comb[2]
        assert abs(ess - 1.0 / (w ** 2).sum()) <= 1e-9 * ess
    np.testing.assert_array_equal(out[0][1], out[1][1])  # every rank finishes identically
    assert G.shard_range(10, 3, 0) == (0, 4) and G.shard_range(10, 3, 2) == (7, 3)
