"""The multi-GPU layer on one GPU: DistAggregation under a world-size-1 NCCL group equals the
single-GPU propagate, and a P-way split of the plan computed shard by shard on the same device
reproduces the unpartitioned result bitwise (the dst-range partition keeps each target's edges
on one owner in the same order)."""
import os
import socket

import numpy as np
import pytest
import torch

import oracle
import synth
from tests.tolerance import check_exact

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_dist_world1_nccl():
    import torch.distributed as dist

    import paper_1903_02428_b200 as pg
    from paper_1903_02428_b200.dist import DistAggregation

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device(DEV))
    try:
        rng = np.random.default_rng(1)
        N, E, F = 5000, 80000, 40
        ei = torch.from_numpy(np.stack([rng.integers(0, N, E), rng.integers(0, N, E)]).astype(np.int64)).to(DEV)
        x = torch.from_numpy(synth.features(N, F, 2, signed=True)).to(DEV)
        da = DistAggregation(ei, N, 1, 0)
        for red in ("sum", "mean", "max"):
            got = da.forward(x, reduce=red)
            ref = pg.pyg_propagate(x, ei, reduce=red, plan=da.plan_full)
            if red == "max":
                check_exact(got[0].cpu().numpy(), ref[0].cpu().numpy())
                check_exact(got[1].cpu().numpy(), ref[1].cpu().numpy())
            else:
                check_exact(got.cpu().numpy(), ref.cpu().numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("P", [2, 3, 8])
def test_partitioned_shards_equal_single(P):
    import paper_1903_02428_b200 as pg
    from paper_1903_02428_b200.dist import partition_rows

    rng = np.random.default_rng(P)
    N, E, F = 3001, 60000, 24
    ei_np = synth.rmat_edges_np(scale=12, E=E, N=N, seed=P)
    ei = torch.from_numpy(ei_np).to(DEV)
    x_np = synth.features(N, F, 3, signed=True)
    x = torch.from_numpy(x_np).to(DEV)
    plan = pg.pyg_plan_build(ei[1], ei[0], N, N)
    ranges, _ = partition_rows(N, P)
    for red in ("sum", "max"):
        full = pg.pyg_propagate(x, ei, reduce=red, plan=plan)
        parts = [pg.pyg_propagate(x, None, n_dst=hi - lo, reduce=red, plan=plan.slice(lo, hi), E=E)
                 for lo, hi in ranges]
        if red == "max":
            check_exact(torch.cat([p[0] for p in parts]).cpu().numpy(), full[0].cpu().numpy())
            check_exact(torch.cat([p[1] for p in parts]).cpu().numpy(), full[1].cpu().numpy())
            ref = oracle.propagate(x_np, ei_np, reduce="max")
            check_exact(full[1].cpu().numpy(), ref[1])
        else:
            check_exact(torch.cat(parts).cpu().numpy(), full.cpu().numpy())
