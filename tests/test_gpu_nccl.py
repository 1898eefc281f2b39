"""The in-library NCCL exchange (gpmppi_planner_attach_comm).

On one GPU: a one-rank communicator runs the sharded tick (reduce -> ncclAllGather ->
finish_kernel) and must reproduce the unsharded planner bit for bit (the rank-order
combine of a single tuple rescales by exp(0) = 1). With >= 2 GPUs (skipped otherwise):
two ranks, one process per GPU, against a single-GPU planner on the same K_total.
The host-side combine and sharding logic is covered on CPU by test_multirank_gloo.py.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_2411_03289_b200 import workloads as W
from tests.helpers import build_pair

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_single_rank_communicator_matches_unsharded():
    import paper_2411_03289_b200 as G
    w = W.CONFIGS["config2"]
    _, a, _, td, _ = build_pair(w, samples=2048)
    _, b, _, _, _ = build_pair(w, samples=2048)
    b.attach_comm(G.nccl_unique_id(), 1, 0)
    assert b.shard() == (0, 2048, 1, 0)
    x = np.array(w.x0)
    for t in range(3):
        da, db = G.StepDiagnostics(), G.StepDiagnostics()
        ca, cb = a.plan_step(x, td, da), b.plan_step(x, td, db)
        np.testing.assert_array_equal(ca, cb)
        np.testing.assert_array_equal(a.nominal_sequence(), b.nominal_sequence())
        np.testing.assert_array_equal(a.sample_costs(), b.sample_costs())
        assert (da.best_cost, da.ess, da.nonfinite_samples) == (db.best_cost, db.ess, db.nonfinite_samples)
        np.testing.assert_array_equal(a.lane_radii(), b.lane_radii())
        x = x + 0.01
    tick_ms, _ = b.bench_device(x, td, 3)
    assert tick_ms.shape == (3,) and (tick_ms > 0).all()
    with pytest.raises(ValueError):
        b.attach_comm(G.nccl_unique_id(), 1, 0)


_WORKER = r"""
import os, sys, numpy as np
sys.path.insert(0, {root!r})
import torch, torch.distributed as dist
rank, world = int(sys.argv[1]), int(sys.argv[2])
torch.cuda.set_device(rank)
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=sys.argv[3])
dist.init_process_group("gloo", rank=rank, world_size=world)
import paper_2411_03289_b200 as G
from paper_2411_03289_b200 import workloads as W
from tests.helpers import build_pair
w = W.CONFIGS["config2"]
_, p, _, td, _ = build_pair(w, samples=3000)
uid = [G.nccl_unique_id() if rank == 0 else None]
dist.broadcast_object_list(uid, src=0)
p.attach_comm(uid[0], world, rank)
x = np.array(w.x0)
out = []
for t in range(2):
    out.append(p.plan_step(x, td))
    x = x + 0.01
np.save(sys.argv[4] + f".{{rank}}.npy", np.array(out + [p.nominal_sequence().reshape(-1)[:2]]))
dist.destroy_process_group()
"""


def test_two_ranks_match_single_gpu(tmp_path):
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs (one process per GPU)")
    import paper_2411_03289_b200 as G
    script = tmp_path / "worker.py"
    script.write_text(_WORKER.format(root=ROOT))
    port = str(29000 + os.getpid() % 1000)
    base = str(tmp_path / "out")
    procs = [subprocess.Popen([sys.executable, str(script), str(r), "2", port, base]) for r in range(2)]
    assert all(p.wait(timeout=600) == 0 for p in procs)
    r0, r1 = np.load(base + ".0.npy"), np.load(base + ".1.npy")
    np.testing.assert_array_equal(r0, r1)  # every rank applies the identical update
    w = W.CONFIGS["config2"]
    _, single, _, td, _ = build_pair(w, samples=3000)
    x = np.array(w.x0)
    ref = []
    for t in range(2):
        ref.append(single.plan_step(x, td))
        x = x + 0.01
    # the two-rank combine sums in a different order: agreement to rounding
    np.testing.assert_allclose(r0[:2], np.array(ref), rtol=0, atol=1e-12)
    del G
