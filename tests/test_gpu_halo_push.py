"""The peer-store halo (pyg_halo_push over CUDA-IPC-mapped peer buffers) with two
ranks sharing the GPU (gloo for the host-side plumbing): over several steps with changing X, every
rank's propagate over [own shard ; pushed halo rows] equals the slice's propagate over the full X
bitwise, for the double-buffered halo blocks."""
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
        from paper_1903_02428_b200.dist import HaloPush, partition_rows

        dev = torch.device("cuda:0")
        torch.cuda.set_device(dev)
        N, E, F = 5000, 120000, 64
        ei = torch.from_numpy(synth.rmat_edges_np(scale=13, E=E, N=N, seed=41)).to(dev)
        plan = pg.pyg_plan_build(ei[1], ei[0], N, N)
        ranges, per = partition_rows(N, world)
        lo, hi = ranges[rank]
        sl = plan.slice(lo, hi)
        hp = HaloPush(sl, N, lo, hi, per, F, world, rank)
        assert hp.host_ordered  # both ranks on cuda:0: steps ordered on the host, no spin-waits
        ok = True
        for step in range(5):
            x = torch.from_numpy(synth.features(N, F, 100 + step, signed=True)).to(dev)
            hp.shard[: hi - lo] = x[lo:hi]
            hplan = hp.exchange()
            for red in ("sum", "max"):
                got = pg.pyg_propagate(hp.xloc, None, n_dst=hi - lo, reduce=red, plan=hplan, E=E)
                ref = pg.pyg_propagate(x, None, n_dst=hi - lo, reduce=red, plan=sl, E=E)
                if red == "max":
                    ok &= bool(torch.equal(got[0], ref[0]) and torch.equal(got[1], ref[1]))
                else:
                    ok &= bool(torch.equal(got, ref))
        q.put((rank, ok, hp.n_halo, int(sum(hp.send_counts))))
        hp.close()
    finally:
        dist.destroy_process_group()


def test_halo_push_two_ranks_one_gpu():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict((r, (ok, nh, ns)) for r, ok, nh, ns in (q.get(timeout=300) for _ in range(world)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        assert res[r][0], f"rank {r}: halo-push propagate differs from the full-X slice"
        assert res[r][1] > 0
    assert res[0][1] == res[1][2] and res[1][1] == res[0][2]


def test_peer_flags_one_process():
    """The device-side step flags of the peer-store halo (pyg_peer_signal / pyg_peer_wait) in ONE
    process on one stream: every wait is enqueued after the signal that satisfies it, so no kernel
    waits on another that might not be resident (the two-process test above orders its steps on the
    host because its ranks share the GPU).  Checks the release store and the wrap-safe comparison."""
    import paper_1903_02428_b200 as pg

    dev = torch.device("cuda:0")
    flags = torch.zeros(6, dtype=torch.int32, device=dev)
    ptrs = [flags.data_ptr() + 4 * i for i in range(6)]
    pg.pyg_peer_signal(ptrs[:3], 7, dev)
    pg.pyg_peer_wait(ptrs[:3], 7, dev)
    pg.pyg_peer_wait(ptrs[:3], 5, dev)  # already past 5
    torch.cuda.synchronize(dev)
    assert flags.tolist() == [7, 7, 7, 0, 0, 0]
    # the step counter wraps: flag 1 (= 2^32 + 1) satisfies a wait for 0xffffffff
    pg.pyg_peer_signal(ptrs[3:], 0xFFFFFFFF, dev)
    pg.pyg_peer_signal(ptrs[3:], 1, dev)
    pg.pyg_peer_wait(ptrs[3:], 0xFFFFFFFF, dev)
    torch.cuda.synchronize(dev)
    assert flags.tolist()[3:] == [1, 1, 1]
