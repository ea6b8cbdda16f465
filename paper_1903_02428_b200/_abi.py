"""ctypes declarations of include/pyg_gs.h (argument marshalling only).

The library is loaded from the package directory (built in-tree by
``paper_1903_02428_b200.build``).  There is NO fallback: if libpygs.so is
missing or fails to load, importing this module raises.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# PYG_LIBPATH selects an experimental build variant of the same library (A/B tuning runs)
LIB_PATH = os.environ.get("PYG_LIBPATH") or os.path.join(HERE, "libpygs.so")

SUM, MEAN, MAX = 0, 1, 2
REDUCE = {"sum": SUM, "add": SUM, "mean": MEAN, "max": MAX}

PHI_CONCAT_XI = 1 << 0
VALIDATE = 1 << 8
FORCE_ATOMIC = 1 << 9
FORCE_SEGMENT = 1 << 10
NO_TMA = 1 << 11

STATUS = {
    0: "PYG_OK", 1: "PYG_ERR_INVALID_ARGUMENT", 2: "PYG_ERR_DIMENSION", 3: "PYG_ERR_INDEX_OUT_OF_BOUNDS",
    4: "PYG_ERR_ALIGNMENT", 5: "PYG_ERR_UNSUPPORTED", 6: "PYG_ERR_CUDA", 7: "PYG_ERR_NCCL", 8: "PYG_ERR_NO_MEMORY",
}


class PygError(RuntimeError):
    def __init__(self, code: int, fn: str, msg: str):
        super().__init__(f"{fn}: {STATUS.get(code, code)}: {msg}")
        self.code = code
        self.status = STATUS.get(code, str(code))


class PlanView(ctypes.Structure):
    _fields_ = [
        ("n_rows", ctypes.c_int64), ("n_cols", ctypes.c_int64), ("E", ctypes.c_int64),
        ("row_offset", ctypes.c_int64), ("rowptr", ctypes.c_void_p), ("col", ctypes.c_void_p),
        ("perm", ctypes.c_void_p), ("perm_is_identity", ctypes.c_int32), ("n_heavy_rows", ctypes.c_int64),
        ("n_heavy_chunks", ctypes.c_int64), ("heavy_threshold", ctypes.c_int32), ("chunk_size", ctypes.c_int32),
        ("col_block", ctypes.c_int64), ("n_col_blocks", ctypes.c_int64),
    ]


class DistPlanInfo(ctypes.Structure):
    _fields_ = [
        ("lo", ctypes.c_int64), ("hi", ctypes.c_int64), ("per", ctypes.c_int64), ("exchange", ctypes.c_int),
        ("n_halo", ctypes.c_int64), ("n_send", ctypes.c_int64), ("n_local_edges", ctypes.c_int64),
        ("col_block", ctypes.c_int64), ("x_shard", ctypes.c_void_p), ("ldx", ctypes.c_int64),
        ("plan", ctypes.c_void_p),
    ]


EXCHANGE = {"auto": 0, "allgather": 1, "halo": 2}

P = ctypes.c_void_p
I64 = ctypes.c_int64
U32 = ctypes.c_uint32
C = ctypes.c_int
SZ = ctypes.c_size_t
PP = ctypes.POINTER(ctypes.c_void_p)

SIGNATURES = {
    "pyg_version": ([], ctypes.c_char_p),
    "pyg_last_error": ([], ctypes.c_char_p),
    "pyg_launch_count": ([], ctypes.c_uint64),
    "pyg_refresh_env": ([], None),
    "pyg_degree": ([P, I64, I64, U32, P, P], C),
    "pyg_plan_workspace_size": ([I64, I64, I64, I64, ctypes.POINTER(SZ)], C),
    "pyg_plan_build": ([P, P, I64, I64, I64, I64, U32, P, SZ, PP, P], C),
    "pyg_plan_suggest_col_block": ([I64, I64, I64, I64, ctypes.POINTER(I64)], C),
    "pyg_atomic_tile_cols": ([I64, I64, I64, ctypes.c_int, ctypes.POINTER(I64)], C),
    "pyg_plan_slice": ([P, I64, I64, PP], C),
    "pyg_plan_passes": ([P, I64, I64, PP], C),
    "pyg_plan_view": ([P, ctypes.POINTER(PlanView)], C),
    "pyg_plan_export": ([P, P, P, P, P], C),
    "pyg_plan_destroy": ([P], None),
    "pyg_halo_workspace_size": ([P, I64, ctypes.POINTER(SZ)], C),
    "pyg_halo_build": ([P, I64, I64, I64, I64, P, SZ, PP, P, ctypes.POINTER(I64), P], C),
    "pyg_ipc_handle": ([P, P, ctypes.POINTER(I64)], C),
    "pyg_ipc_open": ([P, I64, PP], C),
    "pyg_ipc_close": ([P, I64], C),
    "pyg_halo_push": ([P, I64, I64, I64, P, P, P, P, I64, C, P], C),
    "pyg_gather_rows": ([P, I64, I64, I64, P, I64, U32, P, I64, P], C),
    "pyg_workspace_size": ([P, I64, I64, I64, C, U32, ctypes.POINTER(SZ)], C),
    "pyg_scatter": ([P, I64, I64, I64, P, I64, C, U32, P, I64, P, P, P, SZ, P], C),
    "pyg_scatter_backward": ([P, I64, P, I64, I64, I64, C, P, P, P, I64, P], C),
    "pyg_propagate": ([P, I64, I64, I64, P, I64, I64, P, I64, P, I64, I64, P, C, U32, P, I64, P, P, P, SZ, P], C),
    "pyg_propagate_backward": ([P, I64, I64, I64, I64, P, I64, I64, P, C, U32, P, I64, P, P, P, I64, P, I64, P, I64,
                                P, P, P, SZ, P], C),
    "pyg_gcn_norm_workspace_size": ([I64, I64, ctypes.POINTER(SZ)], C),
    "pyg_gcn_norm": ([P, I64, I64, P, U32, P, P, ctypes.POINTER(I64), P, SZ, P], C),
    "pyg_collate": ([I64, P, P, P, I64, I64, U32, P, P, P, P], C),
    "pyg_global_pool": ([P, I64, I64, I64, P, I64, C, P, I64, P, P], C),
    "pyg_gat_transform": ([P, I64, I64, I64, P, I64, I64, I64, P, P, P, I64, P, P, P], C),
    "pyg_dense_transform": ([P, I64, I64, I64, P, I64, I64, P, P, P, I64, P], C),
    "pyg_gcn_layer_workspace_size": ([P, I64, I64, ctypes.POINTER(SZ)], C),
    "pyg_gcn_layer": ([P, I64, I64, I64, P, I64, I64, P, P, P, I64, P, SZ, P], C),
    "pyg_appnp": ([P, I64, I64, I64, P, I64, ctypes.c_float, P, P, I64, P, P, SZ, P], C),
    "pyg_segment_softmax": ([P, I64, I64, I64, P, I64, P, P, I64, P], C),
    "pyg_segment_softmax_backward": ([P, I64, P, I64, I64, I64, I64, P, P, I64, P], C),
    "pyg_gat_propagate": ([P, I64, I64, I64, I64, P, P, I64, I64, ctypes.c_float, P, P, I64, P, P, P, SZ, P], C),
    "pyg_peer_signal": ([P, C, U32, P], C),
    "pyg_peer_wait": ([P, C, U32, P], C),
    "pyg_gat_backward_workspace_size": ([P, P, I64, I64, C, ctypes.POINTER(SZ)], C),
    "pyg_gat_propagate_workspace_size": ([P, I64, I64, ctypes.POINTER(SZ)], C),
    "pyg_gat_backward": ([P, I64, I64, I64, I64, P, P, I64, I64, ctypes.c_float, P, P, P, I64, P, I64, P, P, P, I64, P,
                          P, P, P, SZ, P], C),
    "pyg_dist_unique_id": ([P], C),
    "pyg_dist_init": ([P, C, C, PP], C),
    "pyg_dist_finalize": ([P], None),
    "pyg_dist_plan_build": ([P, P, I64, I64, I64, I64, I64, C, PP, P], C),
    "pyg_dist_plan_info": ([P, ctypes.POINTER(DistPlanInfo)], C),
    "pyg_dist_plan_destroy": ([P], None),
    "pyg_dist_propagate": ([P, P, I64, P, C, U32, P, I64, P, P], C),
    "pyg_dist_propagate_backward": ([P, P, I64, P, C, P, I64, P, I64, P], C),
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python paper_1903_02428_b200/build.py` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (args, res) in SIGNATURES.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    return lib


lib = _load()


def check(code: int, fn: str):
    if code != 0:
        raise PygError(code, fn, lib.pyg_last_error().decode(errors="replace"))


def launch_count() -> int:
    return int(lib.pyg_launch_count())
