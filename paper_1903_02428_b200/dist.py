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


def partition_rows(n: int, world: int):
    """Contiguous destination ranges [lo, hi) per rank, equal shards of ceil(n / world) rows
    (the last ones may be short or empty).  Returns (ranges, rows_per_shard)."""
    per = (n + world - 1) // world if world > 0 else 0
    return [(min(r * per, n), min((r + 1) * per, n)) for r in range(world)], per


def gather_x(x_shard: torch.Tensor, world: int, group=None, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """All-gather equal row shards [per, ld] into [per * world, ld] (rank order = row order)."""
    per = x_shard.shape[0]
    if out is None:
        out = torch.empty((per * world,) + tuple(x_shard.shape[1:]), dtype=x_shard.dtype, device=x_shard.device)
    dist.all_gather_into_tensor(out, x_shard.contiguous(), group=group)
    return out


def reduce_scatter_rows(partial: torch.Tensor, world: int, group=None) -> torch.Tensor:
    """Sum [per * world, F] partials over ranks and return this rank's [per, F] shard."""
    per = partial.shape[0] // world
    out = torch.empty((per,) + tuple(partial.shape[1:]), dtype=partial.dtype, device=partial.device)
    dist.reduce_scatter_tensor(out, partial.contiguous(), group=group)
    return out


def local_edges(edge_index: torch.Tensor, lo: int, hi: int) -> torch.Tensor:
    """In-edges of targets [lo, hi) with targets renumbered to [0, hi - lo), in ascending edge id
    (the order the max tie rule refers to).  Used by the atomic strategy and the tests."""
    m = (edge_index[1] >= lo) & (edge_index[1] < hi)
    sub = edge_index[:, m]
    return torch.stack([sub[0], sub[1] - lo])


class DistAggregation:
    """dst-range partitioned propagate (segment strategy) for one graph shared by all ranks.

    Every rank holds the full edge_index (it is needed once, to build the plan), builds the global
    plan and keeps the slice of its rows; X arrives as this rank's padded shard.
    """

    def __init__(self, edge_index: torch.Tensor, n: int, world: int, rank: int, group=None,
                 col_block: Optional[int] = None, ld: Optional[int] = None):
        import paper_1903_02428_b200 as pg

        self.pg = pg
        self.n, self.world, self.rank, self.group = n, world, rank, group
        self.ranges, self.per = partition_rows(n, world)
        self.lo, self.hi = self.ranges[rank]
        self.E = edge_index.shape[1]
        if col_block is None:
            col_block = pg.pyg_plan_suggest_col_block(self.E, n, n, (ld or 1) * 4) if ld else 0
        self.plan_full = pg.pyg_plan_build(edge_index[1], edge_index[0], n, n, col_block=col_block)
        self.plan = self.plan_full.slice(self.lo, self.hi)
        self.edge_index = edge_index
        self._xbuf = None

    def forward(self, x_shard: torch.Tensor, reduce="sum", out: Optional[torch.Tensor] = None,
                arg_out: Optional[torch.Tensor] = None, edge_weight=None):
        """x_shard: [per, F] (row-strided allowed) -> out [hi - lo, F] (+ global-id arg for max)."""
        F = x_shard.shape[1]
        ld = x_shard.stride(0)
        if self._xbuf is None or self._xbuf.shape[1] != ld:
            self._xbuf = torch.empty((self.per * self.world, ld), dtype=x_shard.dtype, device=x_shard.device)
        full_rows = x_shard.as_strided((x_shard.shape[0], ld), (ld, 1))
        gather_x(full_rows, self.world, self.group, out=self._xbuf)
        x_full = self._xbuf[: self.n, :F]
        return self.pg.pyg_propagate(x_full, None, n_dst=self.hi - self.lo, reduce=reduce, plan=self.plan,
                                     out=out, arg_out=arg_out, E=self.E, edge_weight=edge_weight)
