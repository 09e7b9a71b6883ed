"""ctypes binding of include/gnncg_b200.h (libgnncg_b200.so, built in-tree).

The product path has exactly one compute backend: the sm_100a kernels in this
library.  If the library is missing or no B200 is visible, every call raises --
there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgnncg_b200.so")

i32, i64, u32, u64, f32, sz, vp = C.c_int, C.c_int64, C.c_uint32, C.c_uint64, C.c_float, C.c_size_t, C.c_void_p


class GnncgError(RuntimeError):
    """Base error of the C ABI (status != GNNCG_OK)."""

    status = -1


class TensorError(GnncgError):
    """Shape mismatch -- the reference's gnncg::TensorError (tensor.hpp:13-15)."""

    status = 1


class GraphError(GnncgError):
    """Endpoint out of range -- the reference's gnncg::GraphError (graph.hpp:14-16)."""

    status = 2


class DeviceError(GnncgError):
    """No sm_100 device: the library has no CPU fallback."""

    status = 3


class CudaError(GnncgError):
    status = 4


class WorkspaceError(GnncgError):
    status = 5


class UnsupportedError(GnncgError):
    status = 6


class ArgumentError(GnncgError):
    status = 7


class NcclError(GnncgError):
    """NCCL missing at run time or a collective failed."""

    status = 8


_ERRORS = {c.status: c for c in (TensorError, GraphError, DeviceError, CudaError, WorkspaceError, UnsupportedError,
                                 ArgumentError, NcclError)}


class Index(C.Structure):
    """gnncg_index_t -- one AdjIndex (graph.hpp:19-29) split to SoA."""

    _fields_ = [("num_rows", i64), ("num_edges", i64), ("off", vp), ("nbr", vp), ("eid", vp)]


class Sched(C.Structure):
    """gnncg_sched_t -- edge-balance work items of the unified thread mapping."""

    _fields_ = [("num_items", i64), ("num_split_items", i64), ("num_split_rows", i64), ("chunk", i32),
                ("reserved", i32), ("items", vp), ("split_rows", vp), ("split_first", vp),
                ("gather_off", vp), ("gather_rows", i64)]


P = C.POINTER


class Part(C.Structure):
    """gnncg_part_t -- one rank's share of a destination-row partition (multi-GPU)."""

    _fields_ = [("num_local", i64), ("maxrows", i64), ("nparts", i32), ("rank", i32),
                ("csr_local", P(Index)), ("csr_local_sched", P(Sched)), ("csr_remote", P(Index)),
                ("csr_remote_sched", P(Sched)), ("csc_local", P(Index)), ("csc_local_sched", P(Sched)),
                ("csc_remote", P(Index)), ("csc_remote_sched", P(Sched)), ("bounds", vp)]


_SIGS = {
    "gnncg_last_error": ([], C.c_char_p),
    "gnncg_version": ([], C.c_char_p),
    "gnncg_device_check": ([], i32),
    "gnncg_launch_count": ([], u64),
    "gnncg_cost_counters": ([vp], i32),
    "gnncg_l2_persist": ([sz, P(sz)], i32),
    "gnncg_hot_window_host": ([i64, vp, i64, P(i64)], i32),
    "gnncg_csr_build_workspace": ([i64, i64], sz),
    "gnncg_csr_build": ([i64, i64, vp, vp, vp, vp, vp, vp, sz, vp], i32),
    "gnncg_csr_build_rect": ([i64, i64, i64, vp, vp, vp, vp, vp, vp, sz, vp], i32),
    "gnncg_max_degree": ([P(Index), P(u64), vp], i32),
    "gnncg_partition_rows": ([i64, vp, i32, vp], i32),
    "gnncg_partition_rows_weighted": ([i64, vp, i32, u64, vp], i32),
    "gnncg_gen_chung_lu": ([i64, i64, vp, u64, vp, vp, vp], i32),
    "gnncg_gen_chung_lu_degrees": ([i64, i64, vp, u64, vp, vp], i32),
    "gnncg_gen_chung_lu_rows_workspace": ([i64], sz),
    "gnncg_gen_chung_lu_rows": ([i64, i64, vp, u64, i64, i64, vp, vp, vp, sz, vp], i32),
    "gnncg_sched_build_host": ([i64, vp, i32, P(i64), P(i64), P(i64), vp, vp, vp], i32),
    "gnncg_gemm_workspace": ([i32, i32, i64, i64, i64], sz),
    "gnncg_gemm": ([i32, i32, i64, i64, i64, vp, i64, vp, i64, vp, i64, vp, sz, vp], i32),
    "gnncg_gat_attn_dots": ([i64, i32, i32, vp, vp, vp, vp, vp, vp], i32),
    "gnncg_gat_transform": ([i64, i64, i32, i32, vp, i64, vp, vp, vp, vp, vp, vp, vp, sz, vp], i32),
    "gnncg_gat_workspace": ([P(Sched), P(Sched), i32, i32], sz),
    "gnncg_gat_fwd": ([P(Index), P(Sched), i32, i32, f32, vp, vp, vp, vp, vp, vp, vp, sz, vp], i32),
    "gnncg_gat_bwd_dst": ([P(Index), P(Sched), i32, i32, f32, vp, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp], i32),
    "gnncg_gat_bwd_src": ([P(Index), P(Sched), i32, i32, f32, i64, i64, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp,
                           vp, vp, sz, vp], i32),
    "gnncg_gat_fast_supported": ([i32, i32], i32),
    "gnncg_gat_rec_stride": ([i32], i32),
    "gnncg_gat_bwd_prep": ([i64, i32, i32, vp, vp, vp, vp, vp, vp, vp], i32),
    # Ht, Al, dst_rec, dOut, a_l, a_r, dHt, dAl, dAr, workspace
    "gnncg_gat_bwd_src_fused": ([P(Index), P(Sched), i32, i32, f32, i64, i64, vp, vp, vp, vp, vp, vp, vp, vp, vp,
                                 vp, sz, vp], i32),
    "gnncg_gat_bf16_supported": ([i32, i32], i32),
    "gnncg_pack_bf16": ([i64, vp, vp, vp], i32),
    "gnncg_gat_fwd_bf16": ([P(Index), P(Sched), i32, i32, f32, vp, vp, vp, vp, vp, vp, vp, sz, vp], i32),
    "gnncg_gat_bwd_prep_bf16": ([i64, i32, i32, vp, vp, vp, vp, vp, vp, vp, vp], i32),
    # Ht_bf16, Al, dst_rec, dOut_bf16, a_l, a_r, dHt, dAl, dAr, workspace
    "gnncg_gat_bwd_src_fused_bf16": ([P(Index), P(Sched), i32, i32, f32, i64, i64, vp, vp, vp, vp, vp, vp, vp, vp,
                                      vp, vp, sz, vp], i32),
    "gnncg_gat_attn_grad_workspace": ([i64, i32, i32], sz),
    "gnncg_gat_attn_grad": ([i64, i32, i32, vp, vp, vp, vp, vp, vp, sz, vp], i32),
    "gnncg_edgeconv_fwd": ([P(Index), i32, i64, vp, i64, vp, i64, vp, vp, vp], i32),
    "gnncg_edgeconv_bwd": ([P(Index), P(Index), i32, vp, vp, vp, i64, vp, i64, vp], i32),
    "gnncg_gmm_fwd": ([P(Index), i32, i32, i32, vp, i64, vp, vp, vp, vp], i32),
    "gnncg_gmm_bwd_workspace": ([P(Index), i32, i32], sz),
    "gnncg_gmm_bwd": ([P(Index), P(Index), i32, i32, i32, vp, i64, vp, vp, vp, vp, vp, vp, vp, sz, vp], i32),
    "gnncg_spmm_workspace": ([P(Sched), i32], sz),
    "gnncg_spmm": ([P(Index), P(Sched), i32, vp, vp, vp, i32, vp, vp, sz, vp], i32),
    "gnncg_relu_bwd_workspace": ([i32], sz),
    "gnncg_relu_bwd": ([i64, i32, vp, vp, i32, vp, vp, vp, sz, vp], i32),
    "gnncg_gcn_norm": ([i64, vp, vp, P(Index), P(Index), vp, vp], i32),
    "gnncg_sgd_update": ([i64, f32, vp, vp, vp], i32),
    "gnncg_fill": ([i64, f32, vp, vp], i32),
    "gnncg_sum_workspace": ([], sz),
    "gnncg_sum": ([i64, vp, vp, vp, sz, vp], i32),
    "gnncg_comm_unique_id": ([vp], i32),
    "gnncg_comm_init": ([P(vp), i32, i32, vp], i32),
    "gnncg_comm_init_nccl": ([P(vp), vp], i32),
    "gnncg_comm_destroy": ([vp], i32),
    "gnncg_comm_size": ([vp], i32),
    "gnncg_comm_rank": ([vp], i32),
    "gnncg_comm_allgather": ([vp, vp, vp, i64, vp], i32),
    "gnncg_comm_reduce_scatter": ([vp, vp, vp, i64, vp], i32),
    "gnncg_comm_allreduce": ([vp, vp, i64, vp], i32),
    "gnncg_gat_dist_workspace": ([P(Part), i32, i32], sz),
    # comm, part, heads, f, slope, Ht_all, Al_all, Ar, out, m, d, workspace, stream
    "gnncg_gat_fwd_dist": ([vp, P(Part), i32, i32, f32, vp, vp, vp, vp, vp, vp, vp, sz, vp], i32),
    # comm, part, heads, f, slope, Ht_all, Al_all, Ar, m, d, out, dOut, a_l, a_r, dHt, dAl, dAr,
    # dHt_send, dAl_send, workspace, stream
    "gnncg_gat_bwd_dist": ([vp, P(Part), i32, i32, f32, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp,
                            sz, vp], i32),
}

EXPORTED = tuple(_SIGS)

_lib = None


def lib():
    """Load libgnncg_b200.so (in-tree) and declare every exported signature."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise DeviceError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        for name, (args, res) in _SIGS.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
    return _lib


def last_error() -> str:
    return lib().gnncg_last_error().decode(errors="replace")


def check(rc: int, what: str = ""):
    if rc != 0:
        cls = _ERRORS.get(rc, GnncgError)
        raise cls(f"{what}: {last_error()}" if what else last_error())


def call(name: str, *args):
    check(getattr(lib(), name)(*args), name)


def require_device():
    check(lib().gnncg_device_check(), "gnncg_device_check")


def l2_persist(nbytes: int) -> int:
    """gnncg_l2_persist: opt in to L2-persisting windows over the hottest gathered rows of the
    fused GAT kernels (0 turns it off).  Returns the set-aside granted (clamped to the device)."""
    got = sz()
    call("gnncg_l2_persist", int(nbytes), C.byref(got))
    return int(got.value)


def hot_window(off, n: int) -> int:
    """gnncg_hot_window_host: start row of the n-row window with the most gathers (off = the
    gathered table's per-row read counts as prefix sums, uint64)."""
    import numpy as np

    off = np.ascontiguousarray(off, dtype=np.uint64)
    b = i64()
    call("gnncg_hot_window_host", off.size - 1, off.ctypes.data, int(n), C.byref(b))
    return int(b.value)
