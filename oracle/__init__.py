"""CPU oracle for the gather / phi / scatter-reduce aggregation (arXiv 1903.02428, Eq. 1).

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
module.  The product package ``paper_1903_02428_b200`` never imports it.

This is a ctypes shim over ``oracle.c`` (plain single-threaded C, fp64
accumulation).  Functions take and return numpy arrays; every wrapper only
marshals arguments.  Each C function cites the paper passage it follows.

Parity status per function: every function is
pinned by at least one test in ``tests/test_oracle.py`` against something other
than itself (printed examples, dense brute force, closed forms, invariants).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.c")

SUM, MEAN, MAX = 0, 1, 2
_REDUCE = {"sum": SUM, "add": SUM, "mean": MEAN, "max": MAX}
_ERR = {1: "invalid argument", 2: "dimension error", 3: "index out of bounds"}


class OracleError(RuntimeError):
    def __init__(self, code: int, fn: str):
        super().__init__(f"{fn}: {_ERR.get(code, code)}")
        self.code = code


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (-O2, no OpenMP, no FMA contraction)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "oracle.h"))
    ):
        subprocess.check_call(
            ["gcc", "-O2", "-std=c99", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
             "-o", _SO, _SRC, "-lm"]
        )
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        I = ctypes.c_int64
        C = ctypes.c_int
        sig = {
            "orc_degree": [P, I, I, P],
            "orc_csr": [P, I, I, P, P],
            "orc_scatter": [P, I, I, I, P, I, C, P, P, P],
            "orc_propagate": [P, I, I, I, P, I, I, P, I, P, I, P, C, C, P, P, P],
            "orc_scatter_backward": [P, I, P, I, I, C, P, P],
            "orc_propagate_backward": [P, I, I, I, I, P, I, I, P, C, C, P, P, P, P, P, P, P],
            "orc_gcn_norm": [P, I, I, P, P, P, P, P],
            "orc_collate": [I, P, P, P, P, P, P],
            "orc_global_pool": [P, I, I, P, I, C, P, P],
            "orc_segment_softmax": [P, I, I, P, I, P],
            "orc_dense_transform": [P, I, I, P, I, P, P, P, P],
            "orc_appnp": [P, I, I, P, I, P, I, ctypes.c_double, P],
            "orc_segment_softmax_backward": [P, P, I, I, P, I, P, P],
            "orc_gat": [P, I, I, I, P, P, I, P, I, ctypes.c_double, P, P, P],
            "orc_gat_backward": [P, I, I, I, P, P, I, P, I, ctypes.c_double, P, P, P, P, P, P, P],
        }
        for name, args in sig.items():
            f = getattr(_lib, name)
            f.argtypes = args
            f.restype = ctypes.c_int
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _f32(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float32)


def _i64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.int64)


def _chk(code, fn):
    if code != 0:
        raise OracleError(code, fn)


def _red(reduce):
    return _REDUCE[reduce] if isinstance(reduce, str) else int(reduce)


def _rows(x):
    """(array, n, F, ld) for a 2-D float32 array that may be a strided row view."""
    x = np.asarray(x)
    if x.dtype != np.float32:
        x = x.astype(np.float32)
    if x.ndim != 2:
        raise ValueError("expected a 2-D array")
    if x.strides[1] != 4 or (x.shape[0] > 1 and x.strides[0] % 4):
        x = np.ascontiguousarray(x)
    ld = x.strides[0] // 4 if x.shape[0] > 1 else x.shape[1]
    return x, x.shape[0], x.shape[1], max(ld, x.shape[1])


def degree(index, n):
    index = _i64(index)
    deg = np.zeros(n, np.int64)
    _chk(lib().orc_degree(_p(index), index.size, n, _p(deg)), "degree")
    return deg


def csr(dst, n):
    dst = _i64(dst)
    rowptr = np.zeros(n + 1, np.int64)
    perm = np.zeros(dst.size, np.int64)
    _chk(lib().orc_csr(_p(dst), dst.size, n, _p(rowptr), _p(perm)), "csr")
    return rowptr, perm


def scatter(src, index, dim_size, reduce="sum", with_abs=False):
    src, E, F, lds = _rows(src)
    index = _i64(index)
    if index.size != E:
        raise OracleError(2, "scatter")
    r = _red(reduce)
    out = np.zeros((dim_size, F), np.float32)
    arg = np.zeros((dim_size, F), np.int64) if r == MAX else None
    ab = np.zeros((dim_size, F), np.float64) if with_abs else None
    _chk(lib().orc_scatter(_p(src), E, F, lds, _p(index), dim_size, r, _p(out), _p(arg), _p(ab)),
         "scatter")
    res = [out]
    if r == MAX:
        res.append(arg)
    if with_abs:
        res.append(ab)
    return res[0] if len(res) == 1 else tuple(res)


def propagate(x_src, edge_index, n_dst=None, reduce="sum", edge_weight=None, edge_attr=None,
              x_dst=None, concat_xi=False, with_abs=False):
    """out (and arg for max, abs-sum if with_abs) of Eq. (1) without gamma."""
    x_src, n_src, F, ldx = _rows(x_src)
    edge_index = _i64(edge_index).reshape(2, -1)
    E = edge_index.shape[1]
    if n_dst is None:
        n_dst = n_src
    ldxd = 0
    if x_dst is not None:
        x_dst, nd, Fd, ldxd = _rows(x_dst)
        assert Fd == F and nd >= n_dst
    D = 0
    if edge_attr is not None:
        edge_attr = _f32(edge_attr).reshape(E, -1)
        D = edge_attr.shape[1]
    edge_weight = _f32(edge_weight)
    r = _red(reduce)
    F_out = (F if concat_xi else 0) + F + D
    out = np.zeros((n_dst, F_out), np.float32)
    arg = np.zeros((n_dst, F_out), np.int64) if r == MAX else None
    ab = np.zeros((n_dst, F_out), np.float64) if with_abs else None
    _chk(lib().orc_propagate(_p(x_src), n_src, F, ldx, _p(x_dst), ldxd, n_dst, _p(edge_index), E,
                             _p(edge_attr), D, _p(edge_weight), r, int(bool(concat_xi)), _p(out),
                             _p(arg), _p(ab)), "propagate")
    res = [out]
    if r == MAX:
        res.append(arg)
    if with_abs:
        res.append(ab)
    return res[0] if len(res) == 1 else tuple(res)


def scatter_backward(grad_out, index, reduce="sum", arg=None):
    grad_out = _f32(grad_out)
    dim_size, F = grad_out.shape
    index = _i64(index)
    E = index.size
    r = _red(reduce)
    gs = np.zeros((E, F), np.float32)
    _chk(lib().orc_scatter_backward(_p(grad_out), F, _p(index), E, dim_size, r, _p(_i64(arg)),
                                    _p(gs)), "scatter_backward")
    return gs


def propagate_backward(x_src, edge_index, grad_out, n_dst=None, reduce="sum", edge_weight=None,
                       D=0, concat_xi=False, arg=None, need_x_src=True, need_x_dst=False,
                       need_edge_attr=False, need_edge_weight=False, with_abs=False):
    """dict of gradients of Eq. (1) without gamma (keys x_src, x_dst, edge_attr, edge_weight)."""
    x_src, n_src, F, ldx = _rows(x_src)
    edge_index = _i64(edge_index).reshape(2, -1)
    E = edge_index.shape[1]
    if n_dst is None:
        n_dst = n_src
    grad_out = _f32(grad_out)
    r = _red(reduce)
    F_out = (F if concat_xi else 0) + F + D
    assert grad_out.shape == (n_dst, F_out)
    res = {}
    gxs = np.zeros((n_src, F), np.float32) if need_x_src else None
    gxd = np.zeros((n_dst, F), np.float32) if need_x_dst else None
    gea = np.zeros((E, D), np.float32) if need_edge_attr else None
    gew = np.zeros(E, np.float32) if need_edge_weight else None
    ab = np.zeros((n_src, F), np.float64) if with_abs else None
    _chk(lib().orc_propagate_backward(_p(x_src), n_src, F, ldx, n_dst, _p(edge_index), E, D,
                                      _p(_f32(edge_weight)), r, int(bool(concat_xi)), _p(grad_out),
                                      _p(_i64(arg)), _p(gxs), _p(gxd), _p(gea), _p(gew), _p(ab)),
         "propagate_backward")
    for k, v in (("x_src", gxs), ("x_dst", gxd), ("edge_attr", gea), ("edge_weight", gew),
                 ("abs_x_src", ab)):
        if v is not None:
            res[k] = v
    return res


def gcn_norm(edge_index, N, edge_weight=None):
    """(edge_index' [2 x E'], w' [E']) with remaining self-loops appended."""
    edge_index = _i64(edge_index).reshape(2, -1)
    E = edge_index.shape[1]
    s = np.zeros(E + N, np.int64)
    d = np.zeros(E + N, np.int64)
    w = np.zeros(E + N, np.float32)
    eo = np.zeros(1, np.int64)
    _chk(lib().orc_gcn_norm(_p(edge_index), E, N, _p(_f32(edge_weight)), _p(s), _p(d), _p(w),
                            _p(eo)), "gcn_norm")
    e = int(eo[0])
    return np.stack([s[:e], d[:e]]), w[:e].copy()


def collate(num_nodes, edge_ptr, local_edge_index):
    """(edge_index [2 x Etot], batch [sum N_g], node_ptr [G+1])."""
    num_nodes = _i64(num_nodes)
    edge_ptr = _i64(edge_ptr)
    G = num_nodes.size
    local = _i64(local_edge_index).reshape(2, -1)
    Etot = local.shape[1]
    if G == 0:
        raise OracleError(1, "collate")
    ei = np.zeros((2, Etot), np.int64)
    batch = np.zeros(int(num_nodes.sum()), np.int64)
    node_ptr = np.zeros(G + 1, np.int64)
    _chk(lib().orc_collate(G, _p(num_nodes), _p(edge_ptr), _p(local), _p(ei), _p(batch),
                           _p(node_ptr)), "collate")
    return ei, batch, node_ptr


def global_pool(x, batch, G, reduce="sum"):
    x = _f32(x)
    N, F = x.shape
    r = _red(reduce)
    out = np.zeros((G, F), np.float32)
    arg = np.zeros((G, F), np.int64) if r == MAX else None
    _chk(lib().orc_global_pool(_p(x), N, F, _p(_i64(batch)), G, r, _p(out), _p(arg)),
         "global_pool")
    return (out, arg) if r == MAX else out


def segment_softmax(src, index, n):
    """softmax of src [E x H] within each segment of index."""
    src = _f32(src)
    src = src.reshape(src.shape[0], -1)
    E, H = src.shape
    index = _i64(index)
    out = np.zeros((E, H), np.float32)
    _chk(lib().orc_segment_softmax(_p(src), E, H, _p(index), n, _p(out)), "segment_softmax")
    return out


def segment_softmax_backward(out, grad, index, n, with_abs=False):
    out = _f32(out).reshape(out.shape[0], -1)
    grad = _f32(grad).reshape(out.shape)
    E, H = out.shape
    gs = np.zeros((E, H), np.float32)
    ab = np.zeros((E, H), np.float64) if with_abs else None
    _chk(lib().orc_segment_softmax_backward(_p(out), _p(grad), E, H, _p(_i64(index)), n, _p(gs), _p(ab)),
         "segment_softmax_backward")
    return (gs, ab) if with_abs else gs


def gat(z, s_src, s_dst, edge_index, H, n_dst=None, slope=0.2, with_abs=False):
    """(out [n_dst x H*C], alpha [E x H]) of the GAT aggregation."""
    z = _f32(z)
    n_src, F = z.shape
    C = F // H
    assert C * H == F
    edge_index = _i64(edge_index).reshape(2, -1)
    E = edge_index.shape[1]
    s_src = _f32(s_src).reshape(n_src, H)
    if n_dst is None:
        n_dst = n_src
    s_dst = _f32(s_dst).reshape(n_dst, H)
    out = np.zeros((n_dst, F), np.float32)
    alpha = np.zeros((E, H), np.float32)
    ab = np.zeros((n_dst, F), np.float64) if with_abs else None
    _chk(lib().orc_gat(_p(z), n_src, H, C, _p(s_src), _p(s_dst), n_dst, _p(edge_index), E, float(slope), _p(out),
                       _p(alpha), _p(ab)), "gat")
    return (out, alpha, ab) if with_abs else (out, alpha)


def gat_backward(z, s_src, s_dst, edge_index, H, grad_out, n_dst=None, slope=0.2, with_abs=False):
    """dict(z, s_src, s_dst [, abs_z, abs_s_src, abs_s_dst]) of the GAT aggregation's backward."""
    z = _f32(z)
    n_src, F = z.shape
    C = F // H
    edge_index = _i64(edge_index).reshape(2, -1)
    E = edge_index.shape[1]
    if n_dst is None:
        n_dst = n_src
    g = _f32(grad_out).reshape(n_dst, F)
    gz = np.zeros((n_src, F), np.float32)
    gss = np.zeros((n_src, H), np.float32)
    gsd = np.zeros((n_dst, H), np.float32)
    abz = np.zeros((n_src, F), np.float64) if with_abs else None
    abs_ = np.zeros((n_src, H), np.float64) if with_abs else None
    abd = np.zeros((n_dst, H), np.float64) if with_abs else None
    _chk(lib().orc_gat_backward(_p(z), n_src, H, C, _p(_f32(s_src).reshape(n_src, H)),
                                _p(_f32(s_dst).reshape(n_dst, H)), n_dst, _p(edge_index), E, float(slope), _p(g),
                                _p(gz), _p(gss), _p(gsd), _p(abz), _p(abs_), _p(abd)), "gat_backward")
    res = {"z": gz, "s_src": gss, "s_dst": gsd}
    if with_abs:
        res.update(abs_z=abz, abs_s_src=abs_, abs_s_dst=abd)
    return res


def appnp(h, edge_index, K=10, alpha=0.1, edge_weight=None):
    """APPNP / SGC propagation z_K."""
    h = _f32(h)
    n, F = h.shape
    edge_index = _i64(edge_index).reshape(2, -1)
    out = np.zeros((n, F), np.float32)
    _chk(lib().orc_appnp(_p(h), n, F, _p(edge_index), edge_index.shape[1], _p(_f32(edge_weight)), K, float(alpha),
                         _p(out)), "appnp")
    return out


def dense_transform(x, weight, bias=None, row_scale=None, with_abs=False):
    """Y = diag(row_scale) x weight^T + bias (weight [F_out x F_in])."""
    x = _f32(x)
    weight = _f32(weight)
    M, K = x.shape
    N = weight.shape[0]
    assert weight.shape[1] == K
    y = np.zeros((M, N), np.float32)
    ab = np.zeros((M, N), np.float64) if with_abs else None
    _chk(lib().orc_dense_transform(_p(x), M, K, _p(weight), N, _p(_f32(bias)), _p(_f32(row_scale)), _p(y), _p(ab)),
         "dense_transform")
    return (y, ab) if with_abs else y
