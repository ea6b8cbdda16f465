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


@pytest.mark.parametrize("P,F,tma", [(2, 24, 0), (3, 64, 1), (8, 128, 1), (4, 37, 0)])
def test_halo_plan_equals_slice(P, F, tma, monkeypatch):
    """pyg_halo_build: halo ids = the referenced remote sources (numpy brute force), and the
    propagate over X_loc = [own shard ; pyg_gather_rows(X, halo_ids)] with the rank-local plan is
    bitwise equal to the slice's propagate over the full X (same kernels, same order), for every
    rank of a P-way split emulated on one device; max args stay global and match the oracle."""
    import paper_1903_02428_b200 as pg
    from paper_1903_02428_b200.dist import partition_rows

    monkeypatch.setenv("PYG_SEG_TMA", str(tma))
    N, E = 3001, 60000
    ei_np = synth.rmat_edges_np(scale=12, E=E, N=N, seed=P + 10)
    ei = torch.from_numpy(ei_np).to(DEV)
    x_np = synth.features(N, F, 3, signed=True)
    ld = (F + 3) // 4 * 4
    xb = torch.zeros((N, ld), device=DEV)
    xb[:, :F] = torch.from_numpy(x_np).to(DEV)
    x = xb[:, :F]
    plan = pg.pyg_plan_build(ei[1], ei[0], N, N)
    ranges, per = partition_rows(N, P)
    ref_max = oracle.propagate(x_np, ei_np, reduce="max")
    for lo, hi in ranges:
        sl = plan.slice(lo, hi)
        hp, hids = pg.pyg_halo_build(sl, N, lo, hi, per)
        m = (ei_np[1] >= lo) & (ei_np[1] < hi)
        srcs = np.unique(ei_np[0][m])
        want = srcs[(srcs < lo) | (srcs >= hi)]
        check_exact(hids.cpu().numpy(), want)
        assert hp.view()["n_cols"] == per + want.size
        xl = torch.full((per + want.size, ld), float("nan"), device=DEV)
        xl[: hi - lo] = xb[lo:hi]
        if want.size:
            pg.pyg_gather_rows(xb, hids, out=xl[per:], flags=pg.VALIDATE)
        xloc = xl[:, :F]
        for red in ("sum", "mean", "max"):
            a = pg.pyg_propagate(x, None, n_dst=hi - lo, reduce=red, plan=sl, E=E)
            b = pg.pyg_propagate(xloc, None, n_dst=hi - lo, reduce=red, plan=hp, E=E)
            if red == "max":
                check_exact(b[0].cpu().numpy(), a[0].cpu().numpy())
                check_exact(b[1].cpu().numpy(), a[1].cpu().numpy())
                check_exact(b[1].cpu().numpy(), ref_max[1][lo:hi])
            else:
                check_exact(b.cpu().numpy(), a.cpu().numpy())


def test_halo_errors():
    import paper_1903_02428_b200 as pg

    N = 100
    ei = torch.randint(0, N, (2, 500), device=DEV)
    blocked = pg.pyg_plan_build(ei[1], ei[0], N, N, col_block=30)
    with pytest.raises(pg.PygError):
        pg.pyg_halo_build(blocked.slice(0, 50), N, 0, 50, 50)
    plan = pg.pyg_plan_build(ei[1], ei[0], N, N)
    with pytest.raises(pg.PygError):
        pg.pyg_halo_build(plan.slice(0, 50), N, 0, 50, 40)  # own_rows < own range
    x = torch.zeros((N, 4), device=DEV)
    with pytest.raises(pg.PygError):
        pg.pyg_gather_rows(x, torch.tensor([0, N], device=DEV), flags=pg.VALIDATE)


def test_dist_world1_nccl_halo():
    """DistAggregation(exchange="halo") under a world-size-1 NCCL group (no remote rows: the halo
    is empty and the all-to-all moves nothing) equals the single-GPU propagate."""
    import torch.distributed as dist

    import paper_1903_02428_b200 as pg
    from paper_1903_02428_b200.dist import DistAggregation

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device(DEV))
    try:
        rng = np.random.default_rng(5)
        N, E, F = 4000, 50000, 64
        ei = torch.from_numpy(np.stack([rng.integers(0, N, E), rng.integers(0, N, E)]).astype(np.int64)).to(DEV)
        x = torch.from_numpy(synth.features(N, F, 2, signed=True)).to(DEV)
        da = DistAggregation(ei, N, 1, 0, exchange="halo")
        assert da.n_halo == 0
        for red in ("sum", "max"):
            got = da.forward(x, reduce=red)
            ref = pg.pyg_propagate(x, ei, reduce=red, plan=da.plan_full)
            if red == "max":
                check_exact(got[1].cpu().numpy(), ref[1].cpu().numpy())
                got, ref = got[0], ref[0]
            check_exact(got.cpu().numpy(), ref.cpu().numpy())
    finally:
        dist.destroy_process_group()
