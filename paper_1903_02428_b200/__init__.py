"""paper_1903_02428_b200 -- B200-native gather / phi / scatter-reduce aggregation
(Fey & Lenssen, arXiv 1903.02428, Eq. 1 without gamma).

Thin Python binding over the C ABI of libpygs.so (include/pyg_gs.h): each
function has the C name, marshals torch CUDA tensors into pointers, leading
dimensions and the current stream, allocates outputs/workspace with torch, and
calls the library.  Every step of the path runs in the library's sm_100a
kernels; there is no CPU or PyTorch fallback (importing fails loudly if the
library is missing).
"""
from __future__ import annotations

import ctypes
from typing import Optional

import torch

from . import _abi
from ._abi import (FORCE_ATOMIC, FORCE_SEGMENT, MAX, MEAN, NO_TMA, PHI_CONCAT_XI, SUM, VALIDATE, PygError, check,
                   launch_count, lib)

__all__ = [
    "Plan", "pyg_degree", "pyg_plan_build", "pyg_plan_suggest_col_block", "pyg_atomic_tile_cols", "pyg_scatter", "pyg_scatter_backward", "pyg_propagate",
    "pyg_propagate_backward", "pyg_gcn_norm", "pyg_collate", "pyg_global_pool", "pyg_workspace_size",
    "pyg_halo_build", "pyg_gather_rows", "pyg_ipc_handle", "pyg_ipc_open", "pyg_ipc_close", "pyg_halo_push", "pyg_segment_softmax", "pyg_segment_softmax_backward",
    "pyg_gat_propagate", "pyg_gat_backward", "pyg_gat_backward_workspace_size", "pyg_gat_propagate_workspace_size", "pyg_peer_signal", "pyg_peer_wait", "pyg_appnp", "pyg_dense_transform", "pyg_gcn_layer", "pyg_gat_transform", "launch_count", "PygError", "SUM", "MEAN", "MAX", "PHI_CONCAT_XI", "VALIDATE", "FORCE_ATOMIC",
    "FORCE_SEGMENT", "version", "DistComm", "DistPlan", "pyg_dist_unique_id", "pyg_dist_init", "pyg_dist_plan_build",
    "pyg_dist_propagate", "pyg_dist_propagate_backward",
]


def version() -> str:
    return lib.pyg_version().decode()


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(device=None):
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _red(reduce) -> int:
    return _abi.REDUCE[reduce] if isinstance(reduce, str) else int(reduce)


def _rows(x: torch.Tensor, name: str):
    """(n, F, ld) of a 2-D float32 CUDA tensor whose rows may be strided."""
    if x.dim() != 2:
        raise ValueError(f"{name}: expected 2-D, got {tuple(x.shape)}")
    if x.dtype != torch.float32 or not x.is_cuda:
        raise ValueError(f"{name}: expected a float32 CUDA tensor")
    if x.shape[1] > 1 and x.stride(1) != 1:
        raise ValueError(f"{name}: columns must be contiguous")
    ld = x.stride(0) if x.shape[0] >= 1 else x.shape[1]
    return x.shape[0], x.shape[1], max(ld, x.shape[1])


def _i64(t: torch.Tensor, name: str) -> torch.Tensor:
    if t.dtype != torch.int64 or not t.is_cuda:
        raise ValueError(f"{name}: expected an int64 CUDA tensor")
    return t.contiguous()


def _workspace(nbytes: int, device) -> Optional[torch.Tensor]:
    return torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=device)


class Plan:
    """CSR plan (stable sort of edges by `row_index`).  Owns its workspace."""

    def __init__(self, handle, workspace, parent=None):
        self._h = handle
        self._ws = workspace
        self._parent = parent  # keep the root's workspace alive for slices

    @property
    def handle(self):
        return self._h

    def view(self) -> dict:
        v = _abi.PlanView()
        check(lib.pyg_plan_view(self._h, ctypes.byref(v)), "pyg_plan_view")
        return {f: getattr(v, f) for f, _ in _abi.PlanView._fields_}

    def slice(self, lo: int, hi: int) -> "Plan":
        h = ctypes.c_void_p()
        check(lib.pyg_plan_slice(self._h, lo, hi, ctypes.byref(h)), "pyg_plan_slice")
        return Plan(h, None, parent=self)

    def passes(self, lo: int, hi: int) -> "Plan":
        """View of the source blocks [lo, hi) of a source-blocked plan (pyg_plan_passes)."""
        h = ctypes.c_void_p()
        check(lib.pyg_plan_passes(self._h, lo, hi, ctypes.byref(h)), "pyg_plan_passes")
        return Plan(h, None, parent=self)

    def export(self):
        """(rowptr, col or None, perm) as int64 CUDA tensors (test helper)."""
        v = self.view()
        dev = self._device()
        rowptr = torch.empty(v["n_rows"] + 1, dtype=torch.int64, device=dev)
        check(lib.pyg_plan_export(self._h, _ptr(rowptr), None, None, _stream()), "pyg_plan_export")
        E_p = int(rowptr[-1].item())
        col = torch.empty(E_p, dtype=torch.int64, device=dev) if v["col"] else None
        perm = torch.empty(E_p, dtype=torch.int64, device=dev)
        check(lib.pyg_plan_export(self._h, None, _ptr(col), _ptr(perm), _stream()), "pyg_plan_export")
        return rowptr, col, perm

    def _device(self):
        p = self
        while p._ws is None:
            p = p._parent
        return p._ws.device

    def __del__(self):
        try:
            if self._h:
                lib.pyg_plan_destroy(self._h)
                self._h = None
        except Exception:
            pass


def pyg_halo_build(slice_plan: Plan, n_src: int, own_lo: int, own_hi: int, own_rows: int):
    """Halo of a rank's plan slice (north_star (3)): (halo_plan, halo_ids [n_halo] int64).
    halo_plan gathers from X_loc = [own shard (own_rows rows); X[halo_ids]].  Synchronous."""
    nb = ctypes.c_size_t()
    check(lib.pyg_halo_workspace_size(slice_plan.handle, n_src, ctypes.byref(nb)), "pyg_halo_workspace_size")
    dev = slice_plan._device()
    ws = _workspace(nb.value, dev)
    ids = torch.empty(max(n_src, 1), dtype=torch.int64, device=dev)
    h = ctypes.c_void_p()
    nh = ctypes.c_int64()
    check(lib.pyg_halo_build(slice_plan.handle, n_src, own_lo, own_hi, own_rows, _ptr(ws), nb.value, ctypes.byref(h),
                             _ptr(ids), ctypes.byref(nh), _stream(dev)), "pyg_halo_build")
    return Plan(h, ws, parent=slice_plan), ids[: nh.value]


def pyg_gather_rows(x: torch.Tensor, rows: torch.Tensor, out: Optional[torch.Tensor] = None, flags: int = 0):
    """out[r] = x[rows[r]] (the halo pack)."""
    n_x, F, ldx = _rows(x, "x")
    rows = _i64(rows, "rows")
    n = rows.numel()
    if out is None:
        out = torch.empty((n, F), dtype=torch.float32, device=x.device)
    _, _, ldo = _rows(out, "out") if n > 0 else (0, F, F)
    check(lib.pyg_gather_rows(_ptr(x), n_x, F, ldx, _ptr(rows), n, flags, _ptr(out), ldo, _stream(x.device)),
          "pyg_gather_rows")
    return out


def pyg_plan_suggest_col_block(E: int, n_rows: int, n_cols: int, row_bytes: int) -> int:
    cb = ctypes.c_int64()
    check(lib.pyg_plan_suggest_col_block(E, n_rows, n_cols, row_bytes, ctypes.byref(cb)),
          "pyg_plan_suggest_col_block")
    return cb.value


def pyg_atomic_tile_cols(n_out: int, n_src: int, ncols: int, reduce="sum") -> int:
    """Column-tile width of the atomic strategy (0: one tile); see pyg_gs.h."""
    c = ctypes.c_int64()
    check(lib.pyg_atomic_tile_cols(n_out, n_src, ncols, _red(reduce), ctypes.byref(c)), "pyg_atomic_tile_cols")
    return c.value


def pyg_plan_build(row_index: torch.Tensor, col_index: Optional[torch.Tensor], n_rows: int,
                   n_cols: int = 0, col_block: int = 0) -> Plan:
    """Build a plan: forward plan = (edge_index[1], edge_index[0]); transposed plan for the
    backward = (edge_index[0], edge_index[1]); scatter plan = (index, None).  col_block > 0 builds a
    source-blocked plan (see pyg_plan_suggest_col_block).  Synchronous."""
    row_index = _i64(row_index, "row_index")
    E = row_index.numel()
    if col_index is not None:
        col_index = _i64(col_index, "col_index")
        assert col_index.numel() == E
    nb = ctypes.c_size_t()
    check(lib.pyg_plan_workspace_size(E, n_rows, n_cols, col_block, ctypes.byref(nb)), "pyg_plan_workspace_size")
    ws = _workspace(nb.value, row_index.device)
    h = ctypes.c_void_p()
    check(lib.pyg_plan_build(_ptr(row_index), _ptr(col_index), E, n_rows, n_cols, col_block, 0, _ptr(ws), nb.value,
                             ctypes.byref(h), _stream(row_index.device)), "pyg_plan_build")
    return Plan(h, ws)


def pyg_workspace_size(plan: Optional[Plan], n_out: int, F_out: int, reduce, flags: int = 0,
                       E: Optional[int] = None) -> int:
    """Scratch bytes of a scatter / propagate / backward call; E (edges) sizes the atomic path's hub
    slots and defaults to the plan's edge count."""
    if E is None:
        E = plan.view()["E"] if plan is not None else 0
    nb = ctypes.c_size_t()
    check(lib.pyg_workspace_size(plan.handle if plan else None, E, n_out, F_out, _red(reduce), flags,
                                 ctypes.byref(nb)), "pyg_workspace_size")
    return nb.value


def pyg_degree(index: torch.Tensor, n: int, flags: int = 0) -> torch.Tensor:
    index = _i64(index, "index")
    deg = torch.empty(n, dtype=torch.int32, device=index.device)
    check(lib.pyg_degree(_ptr(index), index.numel(), n, flags, _ptr(deg), _stream(index.device)), "pyg_degree")
    return deg


def pyg_scatter(src: torch.Tensor, index: torch.Tensor, dim_size: int, reduce="sum", plan: Optional[Plan] = None,
                out: Optional[torch.Tensor] = None, arg_out: Optional[torch.Tensor] = None, flags: int = 0,
                workspace: Optional[torch.Tensor] = None):
    """scatter(src, index, reduce).  Returns out, or (out, arg) for max."""
    E, F, lds = _rows(src, "src")
    index = _i64(index, "index")
    r = _red(reduce)
    dev = src.device
    if out is None:
        out = torch.empty((dim_size, F), dtype=torch.float32, device=dev)
    if r == MAX and arg_out is None:
        arg_out = torch.empty((dim_size, F), dtype=torch.int64, device=dev)
    _, _, ldo = _rows(out, "out")
    if workspace is None:
        workspace = _workspace(pyg_workspace_size(plan, dim_size, F, r, flags, E=E), dev)
    check(lib.pyg_scatter(_ptr(src), E, F, lds, _ptr(index), dim_size, r, flags, _ptr(out), ldo, _ptr(arg_out),
                          plan.handle if plan else None, _ptr(workspace), workspace.numel(), _stream(dev)),
          "pyg_scatter")
    return (out, arg_out) if r == MAX else out


def pyg_scatter_backward(grad_out: torch.Tensor, index: torch.Tensor, reduce="sum",
                         arg_out: Optional[torch.Tensor] = None, deg: Optional[torch.Tensor] = None,
                         grad_src: Optional[torch.Tensor] = None):
    dim_size, F, ldg = _rows(grad_out, "grad_out")
    index = _i64(index, "index")
    E = index.numel()
    r = _red(reduce)
    if r == MEAN and deg is None:
        deg = pyg_degree(index, dim_size)
    if grad_src is None:
        grad_src = torch.empty((E, F), dtype=torch.float32, device=grad_out.device)
    _, _, lds = _rows(grad_src, "grad_src")
    check(lib.pyg_scatter_backward(_ptr(grad_out), ldg, _ptr(index), E, F, dim_size, r, _ptr(arg_out), _ptr(deg),
                                   _ptr(grad_src), lds, _stream(grad_out.device)), "pyg_scatter_backward")
    return grad_src


def pyg_propagate(x_src: torch.Tensor, edge_index: Optional[torch.Tensor], n_dst: Optional[int] = None,
                  reduce="sum", edge_weight: Optional[torch.Tensor] = None,
                  edge_attr: Optional[torch.Tensor] = None, x_dst: Optional[torch.Tensor] = None,
                  concat_xi: bool = False, plan: Optional[Plan] = None, out: Optional[torch.Tensor] = None,
                  arg_out: Optional[torch.Tensor] = None, flags: int = 0, E: Optional[int] = None,
                  workspace: Optional[torch.Tensor] = None):
    """Fused gather + phi + reduce of Eq. (1).  Returns out, or (out, arg) for max."""
    n_src, F, ldx = _rows(x_src, "x_src")
    if n_dst is None:
        n_dst = n_src
    if edge_index is not None:
        edge_index = _i64(edge_index, "edge_index")
        assert edge_index.dim() == 2 and edge_index.shape[0] == 2
        E = edge_index.shape[1]
    elif E is None:
        E = plan.view()["E"] if plan is not None else 0
    r = _red(reduce)
    if concat_xi:
        flags |= PHI_CONCAT_XI
    ldxd = 0
    if x_dst is not None:
        _, Fd, ldxd = _rows(x_dst, "x_dst")
        assert Fd == F
    D, lde = 0, 0
    if edge_attr is not None:
        _, D, lde = _rows(edge_attr, "edge_attr")
    F_out = (F if concat_xi else 0) + F + D
    dev = x_src.device
    if out is None:
        out = torch.empty((n_dst, F_out), dtype=torch.float32, device=dev)
    if r == MAX and arg_out is None:
        arg_out = torch.empty((n_dst, F_out), dtype=torch.int64, device=dev)
    _, _, ldo = _rows(out, "out")
    if workspace is None:
        workspace = _workspace(pyg_workspace_size(plan, n_dst, F_out, r, flags, E=E), dev)
    check(lib.pyg_propagate(_ptr(x_src), n_src, F, ldx, _ptr(x_dst), ldxd, n_dst, _ptr(edge_index), E,
                            _ptr(edge_attr), D, lde, _ptr(edge_weight), r, flags, _ptr(out), ldo, _ptr(arg_out),
                            plan.handle if plan else None, _ptr(workspace), workspace.numel(), _stream(dev)),
          "pyg_propagate")
    return (out, arg_out) if r == MAX else out


def pyg_propagate_backward(x_src: Optional[torch.Tensor], edge_index: torch.Tensor, grad_out: torch.Tensor,
                           n_src: Optional[int] = None, F: Optional[int] = None, reduce="sum",
                           edge_weight: Optional[torch.Tensor] = None, D: int = 0, concat_xi: bool = False,
                           arg_out: Optional[torch.Tensor] = None, deg_dst: Optional[torch.Tensor] = None,
                           plan_T: Optional[Plan] = None, need_x_src: bool = True, need_x_dst: bool = False,
                           need_edge_attr: bool = False, need_edge_weight: bool = False, flags: int = 0,
                           grad_x_src: Optional[torch.Tensor] = None):
    """Gradients of pyg_propagate.  Returns a dict."""
    edge_index = _i64(edge_index, "edge_index")
    E = edge_index.shape[1]
    n_dst, F_out, ldg = _rows(grad_out, "grad_out")
    ldx = 0
    if x_src is not None:
        n_src, F, ldx = _rows(x_src, "x_src")
    assert n_src is not None and F is not None
    r = _red(reduce)
    if concat_xi:
        flags |= PHI_CONCAT_XI
    assert F_out == (F if concat_xi else 0) + F + D
    dev = grad_out.device
    if deg_dst is None and (r == MEAN or (concat_xi and need_x_dst)):
        deg_dst = pyg_degree(edge_index[1], n_dst)
    res = {}
    gxs = grad_x_src if grad_x_src is not None else (
        torch.empty((n_src, F), dtype=torch.float32, device=dev) if need_x_src else None)
    gxd = torch.empty((n_dst, F), dtype=torch.float32, device=dev) if (need_x_dst and concat_xi) else None
    gea = torch.empty((E, D), dtype=torch.float32, device=dev) if (need_edge_attr and D > 0) else None
    gew = torch.empty(E, dtype=torch.float32, device=dev) if need_edge_weight else None
    ws = _workspace(pyg_workspace_size(plan_T, n_src, F, SUM, flags, E=E), dev)
    check(lib.pyg_propagate_backward(_ptr(x_src), n_src, F, ldx, n_dst, _ptr(edge_index), E, D, _ptr(edge_weight), r,
                                     flags, _ptr(grad_out), ldg, _ptr(arg_out), _ptr(deg_dst), _ptr(gxs),
                                     gxs.stride(0) if gxs is not None else 0, _ptr(gxd), F, _ptr(gea), D, _ptr(gew),
                                     plan_T.handle if plan_T else None, _ptr(ws), ws.numel(), _stream(dev)),
          "pyg_propagate_backward")
    for k, v in (("x_src", gxs), ("x_dst", gxd), ("edge_attr", gea), ("edge_weight", gew)):
        if v is not None:
            res[k] = v
    return res


def pyg_gcn_norm(edge_index: torch.Tensor, N: int, edge_weight: Optional[torch.Tensor] = None, flags: int = 0):
    """(edge_index' [2 x E'], w' [E']) = GCN normalisation with remaining self-loops. Synchronous."""
    edge_index = _i64(edge_index, "edge_index")
    E = edge_index.shape[1]
    dev = edge_index.device
    nb = ctypes.c_size_t()
    check(lib.pyg_gcn_norm_workspace_size(E, N, ctypes.byref(nb)), "pyg_gcn_norm_workspace_size")
    ws = _workspace(nb.value, dev)
    eo = torch.empty(2 * (E + N), dtype=torch.int64, device=dev)
    wo = torch.empty(E + N, dtype=torch.float32, device=dev)
    e_out = ctypes.c_int64()
    check(lib.pyg_gcn_norm(_ptr(edge_index), E, N, _ptr(edge_weight), flags, _ptr(eo), _ptr(wo),
                           ctypes.byref(e_out), _ptr(ws), nb.value, _stream(dev)), "pyg_gcn_norm")
    e = e_out.value
    return eo[:2 * e].view(2, e), wo[:e]


def pyg_collate(num_nodes: torch.Tensor, edge_ptr: torch.Tensor, local_edge_index: torch.Tensor,
                N_total: Optional[int] = None, flags: int = 0):
    """Block-diagonal mini-batch: (edge_index, batch, node_ptr)."""
    num_nodes = _i64(num_nodes, "num_nodes")
    edge_ptr = _i64(edge_ptr, "edge_ptr")
    local_edge_index = _i64(local_edge_index, "local_edge_index")
    G = num_nodes.numel()
    E_total = local_edge_index.shape[1] if local_edge_index.dim() == 2 else 0
    if N_total is None:
        N_total = int(num_nodes.sum().item()) if G > 0 else 0
    dev = num_nodes.device
    ei = torch.empty((2, E_total), dtype=torch.int64, device=dev)
    batch = torch.empty(N_total, dtype=torch.int64, device=dev)
    node_ptr = torch.empty(G + 1, dtype=torch.int64, device=dev)
    check(lib.pyg_collate(G, _ptr(num_nodes), _ptr(edge_ptr), _ptr(local_edge_index), E_total, N_total, flags,
                          _ptr(ei), _ptr(batch), _ptr(node_ptr), _stream(dev)), "pyg_collate")
    return ei, batch, node_ptr


def pyg_global_pool(x: torch.Tensor, node_ptr: torch.Tensor, reduce="sum"):
    """Global add/mean/max pooling over contiguous graphs."""
    N, F, ldx = _rows(x, "x")
    node_ptr = _i64(node_ptr, "node_ptr")
    G = node_ptr.numel() - 1
    r = _red(reduce)
    out = torch.empty((G, F), dtype=torch.float32, device=x.device)
    arg = torch.empty((G, F), dtype=torch.int64, device=x.device) if r == MAX else None
    check(lib.pyg_global_pool(_ptr(x), N, F, ldx, _ptr(node_ptr), G, r, _ptr(out), F, _ptr(arg), _stream(x.device)),
          "pyg_global_pool")
    return (out, arg) if r == MAX else out


def pyg_segment_softmax(src: torch.Tensor, plan: Plan, dim_size: int, out: Optional[torch.Tensor] = None):
    """softmax of src [E x H] within the segments of the scatter plan's index."""
    E, H, lds = _rows(src, "src")
    if out is None:
        out = torch.empty((E, H), dtype=torch.float32, device=src.device)
    _, _, ldo = _rows(out, "out")
    check(lib.pyg_segment_softmax(_ptr(src), E, H, lds, None, dim_size, plan.handle, _ptr(out), ldo,
                                  _stream(src.device)), "pyg_segment_softmax")
    return out


def pyg_segment_softmax_backward(out: torch.Tensor, grad_out: torch.Tensor, plan: Plan, dim_size: int):
    E, H, ldo = _rows(out, "out")
    _, _, ldg = _rows(grad_out, "grad_out")
    gs = torch.empty((E, H), dtype=torch.float32, device=out.device)
    check(lib.pyg_segment_softmax_backward(_ptr(out), ldo, _ptr(grad_out), ldg, E, H, dim_size, plan.handle, _ptr(gs),
                                           H, _stream(out.device)), "pyg_segment_softmax_backward")
    return gs


def pyg_gat_propagate(z: torch.Tensor, s_src: torch.Tensor, s_dst: torch.Tensor, H: int, plan: Plan,
                      negative_slope: float = 0.2, out: Optional[torch.Tensor] = None,
                      alpha: Optional[torch.Tensor] = None, workspace: Optional[torch.Tensor] = None,
                      row_sums: Optional[torch.Tensor] = None):
    """GAT attention aggregation: (out [n_dst x H*C], alpha [E x H]).
    row_sums [n_dst x H] (optional output): alpha in factored form, alpha / row_sums[dst]."""
    n_src, F, ldz = _rows(z, "z")
    C = F // H
    assert C * H == F
    n_dst = s_dst.shape[0]
    E = plan.view()["E"]
    s_src = s_src.contiguous()
    s_dst = s_dst.contiguous()
    if out is None:
        out = torch.empty((n_dst, F), dtype=torch.float32, device=z.device)
    if alpha is None:
        alpha = torch.empty((E, H), dtype=torch.float32, device=z.device)
    _, _, ldo = _rows(out, "out")
    if workspace is None:
        workspace = _workspace(pyg_gat_propagate_workspace_size(plan, H, C), z.device)
    check(lib.pyg_gat_propagate(_ptr(z), n_src, H, C, ldz, _ptr(s_src), _ptr(s_dst), n_dst, E, negative_slope,
                                plan.handle, _ptr(out), ldo, _ptr(alpha), _ptr(row_sums), _ptr(workspace),
                                workspace.numel(), _stream(z.device)), "pyg_gat_propagate")
    return out, alpha


def pyg_gat_propagate_workspace_size(plan: Plan, H: int, C: int) -> int:
    nb = ctypes.c_size_t()
    check(lib.pyg_gat_propagate_workspace_size(plan.handle, H, C, ctypes.byref(nb)), "pyg_gat_propagate_workspace_size")
    return nb.value


def pyg_gat_backward_workspace_size(plan: Plan, plan_T: Plan, H: int, C: int, row_sums: bool = False) -> int:
    nb = ctypes.c_size_t()
    check(lib.pyg_gat_backward_workspace_size(plan.handle, plan_T.handle, H, C, int(row_sums), ctypes.byref(nb)),
          "pyg_gat_backward_workspace_size")
    return nb.value


def pyg_gat_backward(z: torch.Tensor, s_src: torch.Tensor, s_dst: torch.Tensor, H: int, alpha: torch.Tensor,
                     grad_out: torch.Tensor, plan: Plan, plan_T: Plan, negative_slope: float = 0.2,
                     out: Optional[torch.Tensor] = None, workspace: Optional[torch.Tensor] = None,
                     row_sums: Optional[torch.Tensor] = None):
    """dict(z, s_src, s_dst, logit) gradients of pyg_gat_propagate.  out: the forward output (enables
    the one-pass SDDMM + softmax backward, t_i = g_i . out_i)."""
    n_src, F, ldz = _rows(z, "z")
    C = F // H
    n_dst = s_dst.shape[0]
    E = plan.view()["E"]
    _, _, ldg = _rows(grad_out, "grad_out")
    ldo = _rows(out, "out")[2] if out is not None else 0
    dev = z.device
    gz = torch.empty((n_src, F), dtype=torch.float32, device=dev)
    gss = torch.empty((n_src, H), dtype=torch.float32, device=dev)
    gsd = torch.empty((n_dst, H), dtype=torch.float32, device=dev)
    gl = torch.empty((max(E, 1), H), dtype=torch.float32, device=dev)[:E]
    if workspace is None:
        workspace = _workspace(pyg_gat_backward_workspace_size(plan, plan_T, H, C, row_sums is not None), dev)
    check(lib.pyg_gat_backward(_ptr(z), n_src, H, C, ldz, _ptr(s_src.contiguous()), _ptr(s_dst.contiguous()), n_dst,
                               E, negative_slope, _ptr(alpha), _ptr(row_sums), _ptr(grad_out), ldg, _ptr(out), ldo,
                               plan.handle,
                               plan_T.handle, _ptr(gz), F, _ptr(gss), _ptr(gsd), _ptr(gl), _ptr(workspace),
                               workspace.numel(), _stream(dev)),
          "pyg_gat_backward")
    return {"z": gz, "s_src": gss, "s_dst": gsd, "logit": gl}


def pyg_appnp(h: torch.Tensor, plan: Plan, K: int = 10, alpha: float = 0.1, edge_weight: Optional[torch.Tensor] = None,
              out: Optional[torch.Tensor] = None, scratch: Optional[torch.Tensor] = None,
              workspace: Optional[torch.Tensor] = None):
    """APPNP / SGC K-step propagation z_{k+1} = (1 - alpha) S z_k + alpha h."""
    n, F, ldh = _rows(h, "h")
    dev = h.device
    if out is None:
        out = torch.empty((n, F), dtype=torch.float32, device=dev)
    _, _, ldo = _rows(out, "out")
    if scratch is None and K > 1:
        scratch = torch.empty((n, ldo), dtype=torch.float32, device=dev)[:, :F]
    if workspace is None:  # + E floats: the weights in plan order (streamed by every step)
        extra = plan.view()["E"] * 4 + 256 if edge_weight is not None else 0
        workspace = _workspace(pyg_workspace_size(plan, n, F, SUM) + extra, dev)
    check(lib.pyg_appnp(_ptr(h), n, F, ldh, _ptr(edge_weight), K, alpha, plan.handle, _ptr(out), ldo, _ptr(scratch),
                        _ptr(workspace), workspace.numel(), _stream(dev)), "pyg_appnp")
    return out


def pyg_dense_transform(x: torch.Tensor, weight: torch.Tensor, bias: Optional[torch.Tensor] = None,
                        row_scale: Optional[torch.Tensor] = None, out: Optional[torch.Tensor] = None):
    """Y = diag(row_scale) x weight^T + bias on tcgen05 tensor cores (TF32, fp32 accumulate).
    weight: [F_out x F_in] (torch.nn.Linear layout)."""
    M, K, ldx = _rows(x, "x")
    N, K2, ldw = _rows(weight, "weight")
    assert K2 == K
    if out is None:
        out = torch.empty((M, N), dtype=torch.float32, device=x.device)
    _, _, ldy = _rows(out, "out")
    check(lib.pyg_dense_transform(_ptr(x), M, K, ldx, _ptr(weight), N, ldw, _ptr(bias), _ptr(row_scale), _ptr(out),
                                  ldy, _stream(x.device)), "pyg_dense_transform")
    return out


def pyg_gcn_layer(x: torch.Tensor, weight: torch.Tensor, plan: Plan, bias: Optional[torch.Tensor] = None,
                  out: Optional[torch.Tensor] = None, workspace: Optional[torch.Tensor] = None):
    """GCN layer D^-1/2 (A+I) D^-1/2 x weight^T + bias; `plan` over edges incl. self-loops."""
    n, K, ldx = _rows(x, "x")
    F_out, K2, ldw = _rows(weight, "weight")
    assert K2 == K
    dev = x.device
    if out is None:
        out = torch.empty((n, F_out), dtype=torch.float32, device=dev)
    _, _, ldo = _rows(out, "out")
    if workspace is None:
        nb = ctypes.c_size_t()
        check(lib.pyg_gcn_layer_workspace_size(plan.handle, n, F_out, ctypes.byref(nb)), "pyg_gcn_layer_workspace_size")
        workspace = _workspace(nb.value, dev)
    check(lib.pyg_gcn_layer(_ptr(x), n, K, ldx, _ptr(weight), F_out, ldw, _ptr(bias), plan.handle, _ptr(out), ldo,
                            _ptr(workspace), workspace.numel(), _stream(dev)), "pyg_gcn_layer")
    return out


def pyg_ipc_handle(t: torch.Tensor) -> bytes:
    """72 bytes: the CUDA IPC handle of the allocation holding t (64) + t's byte offset in it (8)."""
    h = ctypes.create_string_buffer(64)
    off = ctypes.c_int64()
    check(lib.pyg_ipc_handle(_ptr(t), h, ctypes.byref(off)), "pyg_ipc_handle")
    return h.raw + off.value.to_bytes(8, "little")


def pyg_ipc_open(handle: bytes) -> int:
    """Map a peer's buffer (from pyg_ipc_handle); returns its device address."""
    p = ctypes.c_void_p()
    off = int.from_bytes(handle[64:72], "little")
    check(lib.pyg_ipc_open(ctypes.c_char_p(handle[:64]), off, ctypes.byref(p)), "pyg_ipc_open")
    return p.value


def pyg_ipc_close(ptr: int, handle: bytes):
    check(lib.pyg_ipc_close(ctypes.c_void_p(ptr), int.from_bytes(handle[64:72], "little")), "pyg_ipc_close")


def pyg_halo_push(x: torch.Tensor, send_rows: torch.Tensor, send_ptr, dst_ptrs, dst_rows, ldd: int):
    """Store x[send_rows[send_ptr[q]:send_ptr[q+1]]] into rows dst_rows[q].. of peer q's buffer dst_ptrs[q]."""
    n_x, F, ldx = _rows(x, "x")
    send_rows = _i64(send_rows, "send_rows") if send_rows.numel() else send_rows
    n = len(dst_ptrs)
    sp = (ctypes.c_int64 * (n + 1))(*send_ptr)
    dp = (ctypes.c_void_p * max(n, 1))(*[p or None for p in dst_ptrs])
    dr = (ctypes.c_int64 * max(n, 1))(*dst_rows)
    check(lib.pyg_halo_push(_ptr(x), n_x, F, ldx, _ptr(send_rows) if send_rows.numel() else None, sp, dp, dr, ldd, n,
                            _stream(x.device)), "pyg_halo_push")


def _flag_array(ptrs):
    return (ctypes.c_void_p * max(len(ptrs), 1))(*[ctypes.c_void_p(p) for p in ptrs])


def pyg_peer_signal(flag_ptrs, value: int, device=None):
    """Release-store value into each device flag (after every earlier write of the stream)."""
    check(lib.pyg_peer_signal(_flag_array(flag_ptrs), len(flag_ptrs), value & 0xFFFFFFFF, _stream(device)),
          "pyg_peer_signal")


def pyg_peer_wait(flag_ptrs, value: int, device=None):
    """Make the stream wait until each device flag reaches value."""
    check(lib.pyg_peer_wait(_flag_array(flag_ptrs), len(flag_ptrs), value & 0xFFFFFFFF, _stream(device)),
          "pyg_peer_wait")


def pyg_gat_transform(x: torch.Tensor, weight: torch.Tensor, att_src: torch.Tensor, att_dst: torch.Tensor, H: int):
    """(z, s_src, s_dst): z = x weight^T on the tensor cores with GAT's per-head attention projections
    fused into the epilogue.  weight [H*C x K]."""
    M, K, ldx = _rows(x, "x")
    N, K2, ldw = _rows(weight, "weight")
    assert K2 == K and N % H == 0
    dev = x.device
    z = torch.empty((M, N), dtype=torch.float32, device=dev)
    ss = torch.empty((M, H), dtype=torch.float32, device=dev)
    sd = torch.empty((M, H), dtype=torch.float32, device=dev)
    check(lib.pyg_gat_transform(_ptr(x), M, K, ldx, _ptr(weight), H, N // H, ldw, _ptr(att_src.contiguous()),
                                _ptr(att_dst.contiguous()), _ptr(z), N, _ptr(ss), _ptr(sd), _stream(dev)),
          "pyg_gat_transform")
    return z, ss, sd


# ---- multi-GPU layer (include/pyg_gs.h "multi-GPU"; north_star (3)) ----------------

def pyg_dist_unique_id() -> bytes:
    """128-byte NCCL unique id (rank 0 makes it; broadcast it over the process group)."""
    buf = ctypes.create_string_buffer(128)
    check(lib.pyg_dist_unique_id(buf), "pyg_dist_unique_id")
    return buf.raw


class DistComm:
    """The library's NCCL communicator (pyg_dist_init / pyg_dist_finalize)."""

    def __init__(self, handle, rank: int, world: int):
        self._h, self.rank, self.world = handle, rank, world

    @property
    def handle(self):
        return self._h

    def close(self):
        if self._h:
            lib.pyg_dist_finalize(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def pyg_dist_init(unique_id: bytes, rank: int, world: int) -> DistComm:
    """Collective: every rank calls it with the same id, its GPU current."""
    h = ctypes.c_void_p()
    buf = ctypes.create_string_buffer(unique_id, 128)
    check(lib.pyg_dist_init(buf, rank, world, ctypes.byref(h)), "pyg_dist_init")
    return DistComm(h, rank, world)


class DistPlan:
    """One rank's share of a dst-range partitioned graph (pyg_dist_plan_build); owns its buffers."""

    def __init__(self, handle, comm: DistComm, F: int):
        self._h, self.comm, self.F = handle, comm, F
        info = _abi.DistPlanInfo()
        check(lib.pyg_dist_plan_info(handle, ctypes.byref(info)), "pyg_dist_plan_info")
        self.lo, self.hi, self.per = info.lo, info.hi, info.per
        self.exchange = {1: "allgather", 2: "halo"}[info.exchange]
        self.n_halo, self.n_send, self.n_local_edges = info.n_halo, info.n_send, info.n_local_edges
        self.col_block, self.ldx = info.col_block, info.ldx
        self._x_ptr = info.x_shard

    @property
    def handle(self):
        return self._h

    def x_shard(self) -> torch.Tensor:
        """[hi - lo, F] view of this rank's rows inside the exchange buffer (write X here)."""
        n = self.hi - self.lo
        if n == 0:
            return torch.empty((0, self.F), dtype=torch.float32, device="cuda")
        # borrow the library's buffer (valid while this DistPlan lives): a strided view over (n, ldx)
        size = (n - 1) * self.ldx + self.F
        return torch.as_strided(_device_view(self._x_ptr, size), (n, self.F), (self.ldx, 1))

    def __del__(self):
        try:
            if self._h:
                lib.pyg_dist_plan_destroy(self._h)
                self._h = None
        except Exception:
            pass


def _device_view(ptr: int, numel: int) -> torch.Tensor:
    """A torch float32 tensor aliasing library-owned device memory (no copy, no ownership)."""
    class _CAI:
        __cuda_array_interface__ = {"shape": (numel,), "typestr": "<f4", "data": (int(ptr), False), "version": 3,
                                    "strides": None, "stream": None}
    return torch.as_tensor(_CAI(), device="cuda")


def pyg_dist_plan_build(comm: DistComm, edge_index: torch.Tensor, n: int, F: int, ld: Optional[int] = None,
                        col_block: int = 0, exchange: str = "auto") -> DistPlan:
    """Collective, synchronous (see the header).  edge_index: the full graph on every rank."""
    edge_index = _i64(edge_index, "edge_index")
    ld = ld or (F + 3) // 4 * 4
    h = ctypes.c_void_p()
    check(lib.pyg_dist_plan_build(comm.handle, _ptr(edge_index), edge_index.shape[1], n, F, ld, col_block,
                                  _abi.EXCHANGE[exchange], ctypes.byref(h), _stream(edge_index.device)),
          "pyg_dist_plan_build")
    return DistPlan(h, comm, F)


def pyg_dist_propagate(plan: DistPlan, x_shard: torch.Tensor, reduce="sum", edge_weight: Optional[torch.Tensor] = None,
                       out: Optional[torch.Tensor] = None, arg_out: Optional[torch.Tensor] = None, flags: int = 0):
    """Rows [lo, hi) of pyg_propagate over the whole graph; returns out (or (out, arg) for max)."""
    n, F, ldx = _rows(x_shard, "x_shard") if x_shard.shape[0] > 0 else (0, plan.F, plan.F)
    r = _red(reduce)
    dev = x_shard.device
    n_own = plan.hi - plan.lo
    if out is None:
        out = torch.empty((n_own, plan.F), dtype=torch.float32, device=dev)
    if r == MAX and arg_out is None:
        arg_out = torch.empty((n_own, plan.F), dtype=torch.int64, device=dev)
    ldo = out.stride(0) if n_own > 0 else plan.F
    check(lib.pyg_dist_propagate(plan.handle, _ptr(x_shard), max(ldx, plan.F), _ptr(edge_weight), r, flags, _ptr(out),
                                 ldo, _ptr(arg_out), _stream(dev)), "pyg_dist_propagate")
    return (out, arg_out) if r == MAX else out


def pyg_dist_propagate_backward(plan: DistPlan, grad_out: torch.Tensor, reduce="sum",
                                edge_weight: Optional[torch.Tensor] = None, arg_out: Optional[torch.Tensor] = None,
                                grad_x: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Rows [lo, hi) of dL/dX (pyg_propagate_backward's grad_x_src over the whole graph)."""
    r = _red(reduce)
    dev = grad_out.device
    n_own = plan.hi - plan.lo
    ldg = grad_out.stride(0) if n_own > 0 else plan.F
    if grad_x is None:
        grad_x = torch.empty((n_own, plan.F), dtype=torch.float32, device=dev)
    lda = arg_out.stride(0) if (arg_out is not None and n_own > 0) else plan.F
    check(lib.pyg_dist_propagate_backward(plan.handle, _ptr(grad_out), ldg, _ptr(edge_weight), r, _ptr(arg_out), lda,
                                          _ptr(grad_x), grad_x.stride(0) if n_own > 0 else plan.F, _stream(dev)),
          "pyg_dist_propagate_backward")
    return grad_x
