"""Multi-GPU aggregation by destination-node ranges (north_star (3)).

One process per GPU (torchrun).  Rank p owns the targets [lo_p, hi_p) and every in-edge of
them, so the BOX of Eq. (1) is completely local: no cross-GPU reduction, results bitwise equal to
one GPU for max/argmax.  The only exchange is the source features: X is sharded by the same
ranges (padded to equal shards of ceil(N/P) rows) and all-gathered over NCCL (NVLink 5 /
NVSwitch) before the local propagate; the output is already sharded like the next layer's X.
The backward computes partial grad_X for every source referenced by the local edges and
reduce-scatters it back to the owners.

The compute runs in libpygs.so (plan slices of one global plan, pyg_propagate /
pyg_propagate_backward); torch.distributed is the plumbing.  The partition and exchange logic
(`partition_rows`, `gather_x`, `reduce_scatter_rows`) is device-agnostic so it is exercised by
world-size-2 gloo tests on CPU.
"""
from __future__ import annotations

from typing import Optional

import torch
import torch.distributed as dist


def _staged(group, *tensors) -> bool:
    """gloo cannot run these collectives on CUDA tensors: stage them through host memory (used to
    exercise the N > 1 path with several processes on one GPU; NCCL is the production backend)."""
    return dist.get_backend(group) == "gloo" and any(t.is_cuda for t in tensors)


def partition_rows(n: int, world: int):
    """Contiguous destination ranges [lo, hi) per rank, equal shards of ceil(n / world) rows
    (the last ones may be short or empty).  Returns (ranges, rows_per_shard)."""
    per = (n + world - 1) // world if world > 0 else 0
    return [(min(r * per, n), min((r + 1) * per, n)) for r in range(world)], per


def aligned_partition(n: int, world: int, block_rows: int):
    """dst ranges whose boundaries are source-block boundaries: per = k * cb with cb <= block_rows,
    so every source block of a plan built with col_block = cb lies inside one rank's shard.
    Returns (ranges, per, cb)."""
    per0 = (n + world - 1) // world if world > 0 else 0
    k = max(1, -(-per0 // max(1, block_rows)))
    cb = max(1, -(-per0 // k))
    per = k * cb
    return [(min(q * per, n), min((q + 1) * per, n)) for q in range(world)], per, cb


class OverlappedGather:
    """The all-gather of the X shards as one broadcast per owner, overlapped with the source-blocked
    propagate (SURVEY 8(e) "Overlap"): the plan's source blocks are aligned with the shards
    (aligned_partition), all P broadcasts are issued at once on NCCL's stream, and the compute stream
    runs owner q's blocks (a pass view) as soon as owner q's rows have landed -- in ascending block
    order, so the result is bitwise the one-GPU result.  Only the first shard's transfer is exposed."""

    def __init__(self, plan_slice, xbuf: torch.Tensor, per: int, cb: int, world: int, rank: int, group=None):
        self.xbuf, self.per, self.world, self.rank, self.group = xbuf, per, world, rank, group
        nb = plan_slice.view()["n_col_blocks"]
        k = per // cb
        self.views = [plan_slice.passes(q * k, min((q + 1) * k, nb)) if q * k < nb else None for q in range(world)]

    def shard(self, q: int) -> torch.Tensor:
        return self.xbuf[q * self.per: (q + 1) * self.per]

    def step(self, compute):
        """compute(view) runs one pass view of the plan on the current stream."""
        if _staged(self.group, self.xbuf):  # gloo test mode: synchronous host-staged broadcasts
            for q in range(self.world):
                h = self.shard(q).cpu()
                dist.broadcast(h, src=q, group=self.group)
                self.shard(q).copy_(h)
            for v in self.views:
                if v is not None:
                    compute(v)
            return
        works = [dist.broadcast(self.shard(q), src=q, group=self.group, async_op=True) for q in range(self.world)]
        for q, v in enumerate(self.views):
            if q != self.rank:
                works[q].wait()  # the compute stream waits for owner q's rows (host not blocked)
            if v is not None:
                compute(v)
        # the rank's own broadcast (issued last for rank world-1) must finish reading the shard before
        # the caller rewrites it for the next step: order the current stream after it too
        works[self.rank].wait()


def gather_x(x_shard: torch.Tensor, world: int, group=None, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """All-gather equal row shards [per, ld] into [per * world, ld] (rank order = row order)."""
    per = x_shard.shape[0]
    if out is None:
        out = torch.empty((per * world,) + tuple(x_shard.shape[1:]), dtype=x_shard.dtype, device=x_shard.device)
    if _staged(group, x_shard, out):
        h = torch.empty(out.shape, dtype=out.dtype)
        dist.all_gather_into_tensor(h, x_shard.contiguous().cpu(), group=group)
        out.copy_(h)
        return out
    dist.all_gather_into_tensor(out, x_shard.contiguous(), group=group)
    return out


def reduce_scatter_rows(partial: torch.Tensor, world: int, group=None) -> torch.Tensor:
    """Sum [per * world, F] partials over ranks and return this rank's [per, F] shard."""
    per = partial.shape[0] // world
    out = torch.empty((per,) + tuple(partial.shape[1:]), dtype=partial.dtype, device=partial.device)
    if _staged(group, partial):
        h = torch.empty(out.shape, dtype=out.dtype)
        dist.reduce_scatter_tensor(h, partial.contiguous().cpu(), group=group)
        out.copy_(h)
        return out
    dist.reduce_scatter_tensor(out, partial.contiguous(), group=group)
    return out


def halo_recv_counts(halo_ids: torch.Tensor, per: int, world: int):
    """Rows this rank receives from each owner: halo ids are ascending, owner = id // per."""
    owners = torch.div(halo_ids.to("cpu"), per, rounding_mode="floor")
    return torch.bincount(owners, minlength=world)[:world].tolist()


def halo_setup(halo_ids: torch.Tensor, lo: int, per: int, world: int, group=None):
    """Plan-time request exchange of the halo: every rank tells each owner which
    of its rows it needs.  Returns (send_rows, send_counts, recv_counts): send_rows are LOCAL row
    ids of this rank's shard, grouped by requesting rank; recv_counts[q] rows arrive from rank q,
    in ascending global id, which is the halo_ids order."""
    recv_counts = halo_recv_counts(halo_ids, per, world)
    dev = halo_ids.device
    cdev = "cpu" if _staged(group, halo_ids) else dev
    rc = torch.tensor(recv_counts, dtype=torch.int64, device=cdev)
    sc = torch.empty_like(rc)
    dist.all_to_all_single(sc, rc, group=group)  # sc[q] = rows rank q wants from me
    send_counts = sc.tolist()
    req = torch.empty(sum(send_counts), dtype=torch.int64, device=cdev)
    dist.all_to_all_single(req, halo_ids.contiguous().to(cdev), send_counts, recv_counts, group=group)
    return (req - lo).to(dev), send_counts, recv_counts


def halo_exchange(x_shard: torch.Tensor, send_rows: torch.Tensor, send_counts, recv_counts, recv_out: torch.Tensor,
                  pack=None, group=None, send_buf: Optional[torch.Tensor] = None):
    """Per-call halo exchange: pack the requested rows (pyg_gather_rows on the GPU) and deliver
    them with one all-to-all into recv_out [n_halo, ld] (contiguous)."""
    if pack is None:
        def pack(x, rows, out):
            return torch.index_select(x, 0, rows, out=out)
    ld = recv_out.shape[1]
    if send_buf is None:
        send_buf = torch.empty((send_rows.numel(), ld), dtype=x_shard.dtype, device=x_shard.device)
    if send_rows.numel() > 0:
        pack(x_shard, send_rows, send_buf)
    if _staged(group, send_buf, recv_out):
        h = torch.empty(recv_out.shape, dtype=recv_out.dtype)
        dist.all_to_all_single(h, send_buf.cpu(), recv_counts, send_counts, group=group)
        recv_out.copy_(h)
        return recv_out
    dist.all_to_all_single(recv_out, send_buf, recv_counts, send_counts, group=group)
    return recv_out


class HaloPush:
    """Peer-store halo exchange (north_star (3)): each owner writes the rows its peers
    requested straight into their X_loc buffers over NVLink with one kernel (pyg_halo_push: gather +
    transfer, no staging buffer, no NCCL), the buffers mapped once with CUDA IPC.  The halo block is
    double-buffered -- X_loc = [own shard (per rows) ; halo A ; halo B], one halo plan per block.
    The steps are ordered on the DEVICE, with no host synchronisation: every rank owns 2 x world
    uint32 flags (mapped into its peers) -- ready[q] = k + 1 once peer q's step-k push into me is
    complete, consumed[q] = k + 1 once peer q finished reading what I pushed at step k -- and
    exchange(k), all enqueued on the current stream, (1) signals consumed = k to the ranks that push
    to me (my step k-1 propagate precedes it on the stream), (2) waits until the ranks I push to
    consumed step k-2 (the last reader of the block being overwritten), (3) pushes, (4) signals
    ready = k + 1 to them, (5) waits for ready = k + 1 from the ranks that push to me.  Every rank
    signals before it waits, so the waits cannot form a cycle.

    Ranks that share one GPU (the one-GPU tests) must not spin on flags another process's kernel
    writes: nothing makes the two kernels co-resident (B200_PROFILING.md; Xid 109 on this driver).
    There the steps are ordered on the HOST instead (stream sync + barrier around the push); the
    flag protocol itself is checked in one process (tests/test_gpu_halo_push.py)."""

    def __init__(self, slice_plan, n: int, lo: int, hi: int, per: int, ld: int, world: int, rank: int, group=None,
                 dtype=torch.float32):
        import paper_1903_02428_b200 as pg

        self.pg, self.world, self.rank, self.group, self.per = pg, world, rank, group, per
        plan_a, ids = pg.pyg_halo_build(slice_plan, n, lo, hi, per)
        self.n_halo = ids.numel()
        plan_b, _ = pg.pyg_halo_build(slice_plan, n, lo, hi, per + self.n_halo)
        self.plans = (plan_a, plan_b)
        self.send_rows, self.send_counts, recv_counts = halo_setup(ids, lo, per, world, group)
        dev = ids.device
        self.xloc = torch.zeros((per + 2 * self.n_halo, ld), dtype=dtype, device=dev)
        # where my block of rows lands in each peer's halo: per + parity * n_halo_q + (rows q gets
        # from owners < me); each rank tells every owner its offset (all-to-all) and its n_halo
        cdev = "cpu" if _staged(group, ids) else dev
        offs = torch.tensor([per + sum(recv_counts[:o]) for o in range(world)], dtype=torch.int64, device=cdev)
        got = torch.empty_like(offs)
        dist.all_to_all_single(got, offs, group=group)
        nh = [None] * world
        dist.all_gather_object(nh, self.n_halo, group=group)
        self.dst_row = [[int(got[q]) + b * int(nh[q]) for q in range(world)] for b in (0, 1)]
        handles = [None] * world
        dist.all_gather_object(handles, pg.pyg_ipc_handle(self.xloc), group=group)
        self.handles = handles
        self.dst = [0 if (q == rank or self.send_counts[q] == 0) else pg.pyg_ipc_open(handles[q]) for q in range(world)]
        self.send_ptr = [0]
        for c in self.send_counts:
            self.send_ptr.append(self.send_ptr[-1] + c)
        # step flags: [ready[world] | consumed[world]] per rank, mapped into every peer
        self.flags = torch.zeros(2 * world, dtype=torch.int32, device=dev)
        fh = [None] * world
        dist.all_gather_object(fh, pg.pyg_ipc_handle(self.flags), group=group)
        self.flag_handles = fh
        self.flag_base = [self.flags.data_ptr() if q == rank else pg.pyg_ipc_open(fh[q]) for q in range(world)]
        uuids = [None] * world
        dist.all_gather_object(uuids, str(torch.cuda.get_device_properties(dev).uuid), group=group)
        self.host_ordered = len(set(uuids)) < world  # ranks share a GPU: no cross-process spin-waits
        self.recv_from = [q for q in range(world) if q != rank and recv_counts[q] > 0]
        self.send_to = [q for q in range(world) if q != rank and self.send_counts[q] > 0]
        torch.cuda.synchronize(dev)
        dist.barrier(group=group)  # every rank's flags are zero before any signal
        self.step = 0

    @property
    def shard(self) -> torch.Tensor:
        """This rank's X rows (write the shard here)."""
        return self.xloc[: self.per]

    def _flag(self, owner: int, kind: int, about: int) -> int:
        """Address of owner's flag `kind` (0 ready, 1 consumed) about peer `about`."""
        return self.flag_base[owner] + 4 * (kind * self.world + about)

    def exchange(self):
        """Push this step's halo rows to every peer and make the stream wait for every peer's push
        into mine, all on the device (see the class notes).  Returns the halo plan to propagate with
        (X_loc = self.xloc); the propagate must be enqueued on the current stream."""
        k, b, me, pg = self.step, self.step & 1, self.rank, self.pg
        dev = self.xloc.device
        if self.host_ordered:
            torch.cuda.current_stream(dev).synchronize()
            dist.barrier(group=self.group)  # every rank's reads of block b (step k - 2) are done
            pg.pyg_halo_push(self.shard, self.send_rows, self.send_ptr, self.dst, self.dst_row[b], self.xloc.stride(0))
            torch.cuda.current_stream(dev).synchronize()
            dist.barrier(group=self.group)  # every push into my halo block has landed
            self.step += 1
            return self.plans[b]
        if k >= 1:  # my step k-1 reads of what they pushed are done (stream order)
            pg.pyg_peer_signal([self._flag(q, 1, me) for q in self.recv_from], k, dev)
        if k >= 2:  # block b was last read at step k-2 by the ranks I push to
            pg.pyg_peer_wait([self._flag(me, 1, q) for q in self.send_to], k - 1, dev)
        pg.pyg_halo_push(self.shard, self.send_rows, self.send_ptr, self.dst, self.dst_row[b], self.xloc.stride(0))
        pg.pyg_peer_signal([self._flag(q, 0, me) for q in self.send_to], k + 1, dev)
        pg.pyg_peer_wait([self._flag(me, 0, q) for q in self.recv_from], k + 1, dev)
        self.step += 1
        return self.plans[b]

    def close(self):
        """Wait until the peers are done with my buffers, then unmap theirs."""
        torch.cuda.synchronize(self.xloc.device)
        dist.barrier(group=self.group)
        for q, p in enumerate(self.dst):
            if p:
                self.pg.pyg_ipc_close(p, self.handles[q])
        self.dst = [0] * self.world
        for q in range(self.world):
            if q != self.rank and self.flag_base[q]:
                self.pg.pyg_ipc_close(self.flag_base[q], self.flag_handles[q])
        self.flag_base = [0] * self.world


def local_edges(edge_index: torch.Tensor, lo: int, hi: int) -> torch.Tensor:
    """In-edges of targets [lo, hi) with targets renumbered to [0, hi - lo), in ascending edge id
    (the order the max tie rule refers to).  Used by the atomic strategy and the tests."""
    m = (edge_index[1] >= lo) & (edge_index[1] < hi)
    sub = edge_index[:, m]
    return torch.stack([sub[0], sub[1] - lo])


def all_to_all_rows(send: torch.Tensor, send_counts, recv: torch.Tensor, recv_counts, group=None):
    """Rows send[soff[q] : soff[q] + send_counts[q]] go to rank q; rows from rank q land in recv in rank
    order (host-staged under gloo)."""
    if _staged(group, send, recv):
        h = torch.empty(recv.shape, dtype=recv.dtype)
        dist.all_to_all_single(h, send.contiguous().cpu(), recv_counts, send_counts, group=group)
        recv.copy_(h)
        return recv
    dist.all_to_all_single(recv, send.contiguous(), recv_counts, send_counts, group=group)
    return recv


class DistAggregation:
    """dst-range partitioned propagate + backward for one graph shared by all ranks.

    backend "nccl" (production): a thin shim over the library's multi-GPU layer -- pyg_dist_init /
    pyg_dist_plan_build / pyg_dist_propagate / pyg_dist_propagate_backward, NCCL inside libpygs
    (include/pyg_gs.h "multi-GPU").  backend "gloo" (test emulation: several ranks on one GPU, or CPU
    collectives): the same algorithm with torch.distributed collectives, host-staged, around the
    library's local kernels.

    Every rank holds the full edge_index (needed once, to build the plans); X arrives as this rank's
    shard of rows [lo, hi).  exchange="allgather": every rank receives every shard (dense graphs);
    "halo": only the referenced remote rows travel and the local buffer is [own shard ; halo rows]
    with rank-local gathered ids (pyg_halo_build); "auto" (nccl) picks per the header's rule.
    Backward: partial dL/dX over every source the local edges reference, then a reduce-scatter
    (all-gather mode) or the reverse halo (halo mode).
    """

    def __init__(self, edge_index: torch.Tensor, n: int, world: int, rank: int, group=None,
                 col_block: Optional[int] = None, ld: Optional[int] = None, exchange: str = "allgather",
                 F: Optional[int] = None, backend: Optional[str] = None, comm=None):
        import paper_1903_02428_b200 as pg

        self.pg = pg
        self.n, self.world, self.rank, self.group = n, world, rank, group
        self.E = edge_index.shape[1]
        self.edge_index = edge_index
        self.backend = backend or (dist.get_backend(group) if dist.is_initialized() else "nccl")
        if col_block is None:
            col_block = pg.pyg_plan_suggest_col_block(self.E, n, n, (ld or 1) * 4) if ld else 0
        self.col_block, self.ld, self.F = col_block, ld, F
        self.exchange = exchange
        self._xbuf = None
        self._loc = None
        if self.backend == "nccl":
            if comm is None:  # the library's own NCCL communicator, id from rank 0 over the process group
                ids = [pg.pyg_dist_unique_id() if rank == 0 else None]
                if world > 1:
                    dist.broadcast_object_list(ids, src=dist.get_global_rank(group, 0) if group is not None else 0,
                                               group=group)
                comm = pg.pyg_dist_init(ids[0], rank, world)
            self.comm = comm
            self.dplan = None
            if F is not None:
                self._build_dist(F)
            return
        if exchange == "auto":
            exchange = self.exchange = "allgather"
        self.ranges, self.per = partition_rows(n, world)
        self.lo, self.hi = self.ranges[rank]
        self.plan_full = pg.pyg_plan_build(edge_index[1], edge_index[0], n, n, col_block=col_block)
        self.plan = self.plan_full.slice(self.lo, self.hi)
        self.n_halo = 0
        if exchange == "halo":
            self.halo_plan, self.halo_ids = pg.pyg_halo_build(self.plan, n, self.lo, self.hi, self.per)
            self.n_halo = self.halo_ids.numel()
            self.send_rows, self.send_counts, self.recv_counts = halo_setup(self.halo_ids, self.lo, self.per, world,
                                                                            group)
            self._sendbuf = None

    # ------------------------------------------------------------------ nccl: the library's layer
    def _build_dist(self, F: int):
        ld = self.ld or (F + 3) // 4 * 4
        self.dplan = self.pg.pyg_dist_plan_build(self.comm, self.edge_index, self.n, F, ld, self.col_block,
                                                 self.exchange)
        self.F, self.ld = F, ld
        self.lo, self.hi, self.per = self.dplan.lo, self.dplan.hi, self.dplan.per
        self.exchange = self.dplan.exchange
        self.n_halo = self.dplan.n_halo

    def x_shard(self, F: Optional[int] = None) -> torch.Tensor:
        """(nccl) this rank's rows inside the library's exchange buffer: writing X there saves a copy."""
        if self.dplan is None:
            self._build_dist(F or self.F)
        return self.dplan.x_shard()

    def local_buffer(self, ld: int, dtype=torch.float32) -> torch.Tensor:
        """(gloo, halo) [per + n_halo, ld] buffer whose first `per` rows are this rank's shard."""
        rows = self.per + self.n_halo
        if self._xbuf is None or tuple(self._xbuf.shape) != (rows, ld):
            self._xbuf = torch.empty((rows, ld), dtype=dtype, device=self.edge_index.device)
        return self._xbuf

    def _forward_halo(self, x_shard, reduce, out, arg_out, edge_weight):
        F = x_shard.shape[1]
        ld = x_shard.stride(0)
        xl = self.local_buffer(ld, x_shard.dtype)
        full_rows = x_shard.as_strided((x_shard.shape[0], ld), (ld, 1))
        if full_rows.data_ptr() != xl.data_ptr():
            xl[: x_shard.shape[0]].copy_(full_rows)
        if self._sendbuf is None or tuple(self._sendbuf.shape) != (self.send_rows.numel(), ld):
            self._sendbuf = torch.empty((self.send_rows.numel(), ld), dtype=xl.dtype, device=xl.device)
        pg = self.pg
        halo_exchange(xl[: self.per], self.send_rows, self.send_counts, self.recv_counts, xl[self.per:],
                      pack=lambda x, rows, o: pg.pyg_gather_rows(x, rows, out=o), group=self.group,
                      send_buf=self._sendbuf)
        x_loc = xl[:, :F]
        return pg.pyg_propagate(x_loc, None, n_dst=self.hi - self.lo, reduce=reduce, plan=self.halo_plan, out=out,
                                arg_out=arg_out, E=self.E, edge_weight=edge_weight)

    def forward(self, x_shard: torch.Tensor, reduce="sum", out: Optional[torch.Tensor] = None,
                arg_out: Optional[torch.Tensor] = None, edge_weight=None):
        """x_shard: [hi - lo, F] (row-strided allowed) -> out [hi - lo, F] (+ global-id arg for max)."""
        if self.backend == "nccl":
            if self.dplan is None:
                self._build_dist(x_shard.shape[1])
            return self.pg.pyg_dist_propagate(self.dplan, x_shard, reduce, edge_weight=edge_weight, out=out,
                                              arg_out=arg_out)
        if self.exchange == "halo":
            return self._forward_halo(x_shard, reduce, out, arg_out, edge_weight)
        F = x_shard.shape[1]
        ld = x_shard.stride(0)
        if self._xbuf is None or self._xbuf.shape[1] != ld:
            self._xbuf = torch.empty((self.per * self.world, ld), dtype=x_shard.dtype, device=x_shard.device)
        full_rows = x_shard.as_strided((x_shard.shape[0], ld), (ld, 1))
        gather_x(full_rows, self.world, self.group, out=self._xbuf)
        x_full = self._xbuf[: self.n, :F]
        return self.pg.pyg_propagate(x_full, None, n_dst=self.hi - self.lo, reduce=reduce, plan=self.plan,
                                     out=out, arg_out=arg_out, E=self.E, edge_weight=edge_weight)

    # ------------------------------------------------------------------ backward
    def _local_edges(self):
        """(gloo) the in-edges of own targets, ascending global id, with sources in the rank's source
        space (global ids padded to per * world, or own-then-halo local ids) and their transposed plan."""
        if self._loc is None:
            pg, ei = self.pg, self.edge_index
            n_own = self.hi - self.lo
            eid = torch.nonzero((ei[1] >= self.lo) & (ei[1] < self.hi)).flatten()
            src, dst = ei[0, eid], ei[1, eid] - self.lo
            if self.exchange == "halo":
                own = (src >= self.lo) & (src < self.hi)
                src = torch.where(own, src - self.lo, self.per + torch.searchsorted(self.halo_ids, src))
                n_src = self.per + self.n_halo
            else:
                n_src = self.per * self.world
            lei = torch.stack([src, dst]).contiguous()
            plan_t = pg.pyg_plan_build(lei[0], lei[1], n_src, n_own)
            deg = pg.pyg_degree(lei[1], n_own)
            self._loc = (eid, lei, n_src, plan_t, deg)
        return self._loc

    def backward(self, grad_out: torch.Tensor, reduce="sum", arg_out: Optional[torch.Tensor] = None,
                 edge_weight=None) -> torch.Tensor:
        """grad_out [hi - lo, F] -> dL/dX rows [hi - lo, F] of this rank (SURVEY 8(e) Backward)."""
        if self.backend == "nccl":
            return self.pg.pyg_dist_propagate_backward(self.dplan, grad_out, reduce, edge_weight=edge_weight,
                                                       arg_out=arg_out)
        pg = self.pg
        eid, lei, n_src, plan_t, deg = self._local_edges()
        n_own, F = grad_out.shape
        w = edge_weight[eid] if edge_weight is not None else None
        arg_l = None
        if reduce == "max":  # global edge ids -> local edge indices (sentinel E -> E_loc)
            j = torch.searchsorted(eid, arg_out.clamp(max=max(self.E - 1, 0)).contiguous())
            arg_l = torch.where(arg_out >= self.E, eid.numel(), j)
        part = pg.pyg_propagate_backward(None, lei, grad_out, n_src=n_src, F=F, reduce=reduce, edge_weight=w,
                                         arg_out=arg_l, deg_dst=deg, plan_T=plan_t)["x_src"]
        if self.exchange != "halo":
            return reduce_scatter_rows(part, self.world, self.group)[:n_own]
        # reverse halo: my halo rows' partials back to their owners; theirs for my rows come back
        rbuf = torch.empty((self.send_rows.numel(), F), dtype=part.dtype, device=part.device)
        all_to_all_rows(part[self.per:], self.recv_counts, rbuf, self.send_counts, self.group)
        add = pg.pyg_scatter(rbuf, self.send_rows, n_own, "sum") if rbuf.shape[0] else None
        g = part[:n_own].clone()
        if add is not None:
            g += add
        return g
