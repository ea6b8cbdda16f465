"""N > 1 path on CPU: world-size-2 gloo processes run the dst-range partition and the exchange
(all-gather of X shards, reduce-scatter of partial grad_X) of paper_1903_02428_b200.dist, with the
oracle standing in for the local GPU kernel.  The partitioned result must equal the single-process
oracle: bitwise for sum/mean/max/argmax (each target's in-edges stay in ascending edge order on
its owner), within tolerance for the reduce-scattered gradient."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, N, F, seed, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import synth
        from paper_1903_02428_b200.dist import gather_x, local_edges, partition_rows, reduce_scatter_rows

        rng = np.random.default_rng(seed)
        E = 6 * N
        ei = np.stack([rng.integers(0, N, E), rng.integers(0, N, E)]).astype(np.int64)
        x = synth.features(N, F, seed, signed=True)
        g = synth.features(N, F, seed + 1, signed=True)
        ranges, per = partition_rows(N, world)
        lo, hi = ranges[rank]
        shard = torch.zeros((per, F))
        shard[: hi - lo] = torch.from_numpy(x[lo:hi])
        xfull = gather_x(shard, world)[:N].numpy()
        res = {"x_equal": bool(np.array_equal(xfull, x))}
        tei = torch.from_numpy(ei)
        loc = local_edges(tei, lo, hi).numpy()
        gid = torch.nonzero((tei[1] >= lo) & (tei[1] < hi)).flatten().numpy()
        outs = {}
        for red in ("sum", "mean", "max"):
            r = oracle.propagate(xfull, loc, n_dst=hi - lo, reduce=red)
            if red == "max":
                o, a = r
                a = np.where(a == loc.shape[1], E, gid[np.minimum(a, max(loc.shape[1] - 1, 0))] if gid.size else E)
                outs[red] = (o, a)
            else:
                outs[red] = r
        # backward: partial grad_X over all sources from the local edges, reduce-scattered to owners
        part = oracle.propagate_backward(xfull, loc, g[lo:hi], n_dst=hi - lo, reduce="mean")["x_src"]
        padded = torch.zeros((per * world, F))
        padded[:N] = torch.from_numpy(part)
        mine = reduce_scatter_rows(padded, world)[: hi - lo].numpy()
        res.update(lo=lo, hi=hi, outs=outs, grad=mine)
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("N", [37, 1000])
def test_dst_partition_equals_single_process(N):
    import oracle
    import synth
    from tests.tolerance import check_close

    world, F, seed = 2, 5, 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, N, F, seed, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(seed)
    E = 6 * N
    ei = np.stack([rng.integers(0, N, E), rng.integers(0, N, E)]).astype(np.int64)
    x = synth.features(N, F, seed, signed=True)
    g = synth.features(N, F, seed + 1, signed=True)
    full = {red: oracle.propagate(x, ei, reduce=red) for red in ("sum", "mean", "max")}
    gfull = oracle.propagate_backward(x, ei, g, reduce="mean", with_abs=True)
    for r in range(world):
        res = results[r]
        lo, hi = res["lo"], res["hi"]
        assert res["x_equal"]
        for red in ("sum", "mean"):
            assert np.array_equal(res["outs"][red], full[red][lo:hi]), red
        assert np.array_equal(res["outs"]["max"][0], full["max"][0][lo:hi])
        assert np.array_equal(res["outs"]["max"][1], full["max"][1][lo:hi])
        check_close(res["grad"], gfull["x_src"][lo:hi], abs_sum=gfull["abs_x_src"][lo:hi])


def test_partition_rows_cover_and_pad():
    from paper_1903_02428_b200.dist import partition_rows

    for n, w in ((10, 3), (232965, 8), (5, 8), (0, 2)):
        ranges, per = partition_rows(n, w)
        assert len(ranges) == w
        assert ranges[0][0] == 0 and ranges[-1][1] == n
        for (a, b), (c, d) in zip(ranges, ranges[1:]):
            assert b == c and b - a <= per


def _halo_worker(rank, world, port, N, F, seed, q):
    """Halo exchange (north_star (3)) with the oracle as the local kernel: only the
    remote rows the local edges reference travel; the local propagate over [own shard ; halo]
    with rank-local source ids must equal the single-process result bitwise."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import synth
        from paper_1903_02428_b200.dist import halo_exchange, halo_setup, local_edges, partition_rows

        ei = synth.rmat_edges_np(scale=10, E=8 * N, N=N, seed=seed)
        E = ei.shape[1]
        x = synth.features(N, F, seed, signed=True)
        ranges, per = partition_rows(N, world)
        lo, hi = ranges[rank]
        tei = torch.from_numpy(ei)
        loc = local_edges(tei, lo, hi).numpy()
        gid = torch.nonzero((tei[1] >= lo) & (tei[1] < hi)).flatten().numpy()
        # halo ids (here: numpy; on the GPU: pyg_halo_build)
        src = np.unique(loc[0])
        halo = src[(src < lo) | (src >= hi)]
        send_rows, sc, rc = halo_setup(torch.from_numpy(halo), lo, per, world)
        ld = F + 3  # padded rows travel whole
        xl = torch.zeros((per + halo.size, ld))
        xl[: hi - lo, :F] = torch.from_numpy(x[lo:hi])
        halo_exchange(xl[:per], send_rows, sc, rc, xl[per:])
        res = {"halo_rows_equal": bool(np.array_equal(xl[per:, :F].numpy(), x[halo])),
               "n_halo": int(halo.size), "sent": int(sum(sc)), "lo": lo, "hi": hi}
        # rank-local source ids: own j -> j - lo, halo h -> per + h
        m = np.full(N, -1, np.int64)
        m[lo:hi] = np.arange(hi - lo)
        m[halo] = per + np.arange(halo.size)
        lei = np.stack([m[loc[0]], loc[1]])
        assert (lei[0] >= 0).all()
        xloc = np.ascontiguousarray(xl[:, :F].numpy())
        outs = {}
        for red in ("sum", "mean", "max"):
            r = oracle.propagate(xloc, lei, n_dst=hi - lo, reduce=red)
            if red == "max":
                o, a = r
                a = np.where(a == lei.shape[1], E, gid[np.minimum(a, max(lei.shape[1] - 1, 0))] if gid.size else E)
                outs[red] = (o, a)
            else:
                outs[red] = r
        res["outs"] = outs
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("N", [64, 2000])
def test_halo_exchange_equals_single_process(N):
    import oracle
    import synth

    world, F, seed = 2, 6, 11
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_halo_worker, args=(r, world, port, N, F, seed, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ei = synth.rmat_edges_np(scale=10, E=8 * N, N=N, seed=seed)
    x = synth.features(N, F, seed, signed=True)
    full = {red: oracle.propagate(x, ei, reduce=red) for red in ("sum", "mean", "max")}
    # what each rank received is what the other was asked to send
    assert results[0]["n_halo"] == results[1]["sent"] and results[1]["n_halo"] == results[0]["sent"]
    for r in range(world):
        res = results[r]
        lo, hi = res["lo"], res["hi"]
        assert res["halo_rows_equal"]
        assert 0 < res["n_halo"] < N - (hi - lo) + 1
        for red in ("sum", "mean"):
            assert np.array_equal(res["outs"][red], full[red][lo:hi]), red
        assert np.array_equal(res["outs"]["max"][0], full["max"][0][lo:hi])
        assert np.array_equal(res["outs"]["max"][1], full["max"][1][lo:hi])


def test_aligned_partition():
    from paper_1903_02428_b200.dist import aligned_partition

    for n, w, b in ((232965, 8, 21179), (10, 3, 2), (6001, 2, 1100), (5, 8, 100)):
        ranges, per, cb = aligned_partition(n, w, b)
        assert per % cb == 0 and cb <= max(b, 1) and per * w >= n
        assert ranges[0][0] == 0 and ranges[-1][1] == n
