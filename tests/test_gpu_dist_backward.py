"""The dst-range partitioned propagate AND its backward (SURVEY 8(e) "Backward"; "both for
forward and backward passes") with two ranks sharing the GPU (dist.DistAggregation, backend gloo:
the exchange is host-staged, every local step runs in libpygs), against the ORACLE over the whole
graph: each rank's output rows and its rows of dL/dX.  Both exchanges: all-gather (backward =
reduce-scatter of the partial gradients) and halo (backward = the reverse halo).  Weighted sum /
mean, and max routed through the forward's (global) argmax."""
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


def _worker(rank, world, port, exchange, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import synth
        from paper_1903_02428_b200.dist import DistAggregation
        from tests.tolerance import check_close, check_exact

        dev = torch.device("cuda:0")
        torch.cuda.set_device(dev)
        N, E, F = 3001, 40000, 24
        ei_np = synth.rmat_edges_np(scale=12, E=E, N=N, seed=31)
        ei = torch.from_numpy(ei_np).to(dev)
        da = DistAggregation(ei, N, world, rank, exchange=exchange, backend="gloo")
        lo, hi, per = da.lo, da.hi, da.per
        w_np = (np.random.default_rng(32).random(E) + 0.5).astype(np.float32)
        w = torch.from_numpy(w_np).to(dev)
        g_np = synth.features(N, F, 33, signed=True)
        msgs = []
        for red in ("sum", "mean", "max"):
            x_np = synth.features(N, F, 34, signed=(red == "max"))
            shard = torch.zeros((per, F), device=dev)
            shard[: hi - lo] = torch.from_numpy(x_np[lo:hi]).to(dev)
            wr = None if red == "max" else w
            wr_np = None if red == "max" else w_np
            res = da.forward(shard, reduce=red, edge_weight=wr)
            ref = oracle.propagate(x_np, ei_np, reduce=red, edge_weight=wr_np)
            g = torch.from_numpy(g_np[lo:hi]).to(dev)
            try:
                if red == "max":
                    check_exact(res[0].cpu().numpy(), ref[0][lo:hi])
                    check_exact(res[1].cpu().numpy(), ref[1][lo:hi])
                    gx = da.backward(g, reduce="max", arg_out=res[1])
                    gref = oracle.propagate_backward(x_np, ei_np, g_np, reduce="max", arg=ref[1])
                    bound = np.abs(gref["x_src"]) + 16 * np.abs(g_np).max()
                else:
                    check_close(res.cpu().numpy(), ref[lo:hi])
                    gx = da.backward(g, reduce=red, edge_weight=wr)
                    gref = oracle.propagate_backward(x_np, ei_np, g_np, reduce=red, edge_weight=wr_np, with_abs=True)
                    bound = gref["abs_x_src"]
                check_close(gx.cpu().numpy(), gref["x_src"][lo:hi], abs_sum=bound[lo:hi], what=f"grad {red}")
            except AssertionError as e:
                msgs.append(f"rank {rank} {exchange} {red}: {e}")
        q.put((rank, msgs, da.n_halo))
    except Exception as e:  # surface worker errors in the parent
        q.put((rank, [f"rank {rank} crashed: {e!r}"], -1))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("exchange", ["allgather", "halo"])
def test_two_ranks_forward_backward_vs_oracle(exchange):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, exchange, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    msgs = [m for _, ms, _ in res for m in ms]
    assert not msgs, "\n".join(msgs)
    if exchange == "halo":
        assert all(nh > 0 for _, _, nh in res)  # remote rows really travel
