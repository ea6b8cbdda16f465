"""dist.OverlappedGather (SURVEY 8(e) "Overlap"): shard-aligned source blocks, one broadcast per
owner, each owner's block passes run after its rows land -- with two ranks sharing the GPU (gloo
stages the broadcasts through host memory), every rank's output equals the whole plan's slice on
the full X bitwise (sum, mean, max + arg), because the passes keep ascending block order."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1903_02428_b200 as pg
        import synth
        from paper_1903_02428_b200.dist import OverlappedGather, aligned_partition

        dev = torch.device("cuda:0")
        torch.cuda.set_device(dev)
        N, E, F = 6001, 90000, 40
        rng = np.random.default_rng(7)
        ei = torch.from_numpy(np.stack([rng.integers(0, N, E), rng.integers(0, N, E)]).astype(np.int64)).to(dev)
        ranges, per, cb = aligned_partition(N, world, 1100)
        assert per % cb == 0
        plan = pg.pyg_plan_build(ei[1], ei[0], N, N, col_block=cb)
        lo, hi = ranges[rank]
        sl = plan.slice(lo, hi)
        xbuf = torch.zeros((per * world, F), device=dev)
        ovg = OverlappedGather(sl, xbuf, per, cb, world, rank)
        ok = True
        for step, red in enumerate(("sum", "mean", "max")):
            x = torch.from_numpy(synth.features(N, F, 50 + step, signed=True)).to(dev)
            xbuf.zero_()
            ovg.shard(rank)[: hi - lo] = x[lo:hi]
            out = torch.empty((hi - lo, F), device=dev)
            arg = torch.empty((hi - lo, F), dtype=torch.int64, device=dev) if red == "max" else None
            ovg.step(lambda v: pg.pyg_propagate(xbuf[:N], None, n_dst=hi - lo, reduce=red, plan=v, E=E, out=out,
                                                arg_out=arg))
            ref = pg.pyg_propagate(x, None, n_dst=hi - lo, reduce=red, plan=sl, E=E)
            if red == "max":
                ok &= bool(torch.equal(out, ref[0]) and torch.equal(arg, ref[1]))
            else:
                ok &= bool(torch.equal(out, ref))
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def test_overlapped_gather_two_ranks_one_gpu():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0] and res[1]
