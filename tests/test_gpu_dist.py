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
from tests.tolerance import check_close, check_exact

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _graph(N, E, seed):
    return synth.rmat_edges_np(scale=12, E=E, N=N, seed=seed)


@pytest.mark.parametrize("col_block", [0, 700])
@pytest.mark.parametrize("red", ["sum", "mean", "max"])
def test_capi_dist_world1_vs_oracle(col_block, red):
    """The C-ABI multi-GPU layer (pyg_dist_init over NCCL, pyg_dist_plan_build, pyg_dist_propagate,
    pyg_dist_propagate_backward) at world size 1, forward and backward against the oracle over the
    whole graph (unblocked and source-blocked plans; weighted for sum / mean)."""
    import paper_1903_02428_b200 as pg

    N, E, F = 3001, 40000, 40
    ei_np = _graph(N, E, 21)
    ei = torch.from_numpy(ei_np).to(DEV)
    x_np = synth.features(N, F, 22, signed=(red == "max"))
    g_np = synth.features(N, F, 23, signed=True)
    w_np = None if red == "max" else (np.random.default_rng(24).random(E) + 0.5).astype(np.float32)
    w = torch.from_numpy(w_np).to(DEV) if w_np is not None else None
    comm = pg.pyg_dist_init(pg.pyg_dist_unique_id(), 0, 1)
    dp = pg.pyg_dist_plan_build(comm, ei, N, F, ld=44, col_block=col_block)
    assert (dp.lo, dp.hi, dp.exchange, dp.n_local_edges) == (0, N, "allgather", E)
    xs = dp.x_shard()  # write X straight into the library's exchange buffer
    xs.copy_(torch.from_numpy(x_np))
    res = pg.pyg_dist_propagate(dp, xs, red, edge_weight=w)
    ref = oracle.propagate(x_np, ei_np, reduce=red, edge_weight=w_np)
    if red == "max":
        check_exact(res[0].cpu().numpy(), ref[0])
        check_exact(res[1].cpu().numpy(), ref[1])
        arg = res[1]
        gref = oracle.propagate_backward(x_np, ei_np, g_np, reduce="max", arg=ref[1])
        bound = np.abs(gref["x_src"]) + 16 * np.abs(g_np).max()
    else:
        check_close(res.cpu().numpy(), ref)
        arg = None
        gref = oracle.propagate_backward(x_np, ei_np, g_np, reduce=red, edge_weight=w_np, with_abs=True)
        bound = gref["abs_x_src"]
    # a copy from another buffer (x_shard not the library's) gives the same result
    res2 = pg.pyg_dist_propagate(dp, torch.from_numpy(x_np).to(DEV), red, edge_weight=w)
    check_exact((res2[0] if red == "max" else res2).cpu().numpy(), (res[0] if red == "max" else res).cpu().numpy())
    gx = pg.pyg_dist_propagate_backward(dp, torch.from_numpy(g_np).to(DEV), red, edge_weight=w, arg_out=arg)
    check_close(gx.cpu().numpy(), gref["x_src"], abs_sum=bound)
    del dp
    comm.close()


def test_capi_dist_errors():
    import paper_1903_02428_b200 as pg

    comm = pg.pyg_dist_init(pg.pyg_dist_unique_id(), 0, 1)
    ei = torch.randint(0, 100, (2, 500), device=DEV)
    with pytest.raises(pg.PygError) as e:  # the halo needs an unblocked plan
        pg.pyg_dist_plan_build(comm, ei, 100, 8, col_block=30, exchange="halo")
    assert e.value.status == "PYG_ERR_UNSUPPORTED"
    with pytest.raises(pg.PygError) as e:
        pg.pyg_dist_plan_build(comm, ei, 100, 8, ld=6)
    assert e.value.status == "PYG_ERR_DIMENSION"
    dp = pg.pyg_dist_plan_build(comm, ei, 100, 8)
    with pytest.raises(pg.PygError) as e:  # null x / out
        pg._abi.check(pg.lib.pyg_dist_propagate(dp.handle, None, 8, None, 2, 0, None, 8, None, None),
                      "pyg_dist_propagate")
    assert e.value.status == "PYG_ERR_INVALID_ARGUMENT"
    with pytest.raises(pg.PygError) as e:  # rank outside [0, world)
        pg.pyg_dist_init(pg.pyg_dist_unique_id(), 1, 1)
    assert e.value.status == "PYG_ERR_INVALID_ARGUMENT"
    del dp
    comm.close()


def test_dist_world1_nccl():
    """DistAggregation (backend nccl = the library's layer) under a world-size-1 torch NCCL group."""
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
        for exchange in ("allgather", "halo", "auto"):
            da = DistAggregation(ei, N, 1, 0, exchange=exchange)
            plan = pg.pyg_plan_build(ei[1], ei[0], N, N)
            for red in ("sum", "mean", "max"):
                got = da.forward(x, reduce=red)
                ref = pg.pyg_propagate(x, ei, reduce=red, plan=plan)
                if red == "max":
                    check_exact(got[0].cpu().numpy(), ref[0].cpu().numpy())
                    check_exact(got[1].cpu().numpy(), ref[1].cpu().numpy())
                else:
                    check_exact(got.cpu().numpy(), ref.cpu().numpy())
            assert da.exchange == "allgather" and da.n_halo == 0  # one rank: nothing is remote
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
