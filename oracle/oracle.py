"""oracle/oracle.py -- TEST INFRASTRUCTURE ONLY.

ctypes bindings for the CPU restatement (``liboracle.so``, see oracle.cpp for the
reference file:line each function follows) and for the reference's own graph /
tensor code (``_ref/libgnncg_ref.so``, built by oracle/Makefile from
/root/reference/proj/src).  Only tests/, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of bench.py may import this module.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_ORC = None
_REF = None

u64 = C.c_uint64
i32 = C.c_int
f64 = C.c_double
f32 = C.c_float
vp = C.c_void_p


def _p(a):
    return None if a is None else a.ctypes.data_as(vp)


def lib():
    global _ORC
    if _ORC is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            raise RuntimeError(f"oracle not built: {path} (run `make -C oracle`)")
        _ORC = C.CDLL(path)
        _ORC.orc_num_threads.restype = i32
        for n in ("orc_gat_attn_flops_naive", "orc_gat_attn_flops_reorg", "orc_gat_io_unfused", "orc_gat_io_fused"):
            getattr(_ORC, n).restype = u64
    return _ORC


def ref_available() -> bool:
    return os.path.exists(os.path.join(_HERE, "_ref", "libgnncg_ref.so"))


def ref():
    """The reference's own graph.cpp/tensor.cpp behind ref_shim.cpp."""
    global _REF
    if _REF is None:
        path = os.path.join(_HERE, "_ref", "libgnncg_ref.so")
        if not os.path.exists(path):
            raise RuntimeError(f"reference shim not built: {path}")
        _REF = C.CDLL(path)
        _REF.ref_graph_new.restype = vp
        _REF.ref_graph_synthetic.restype = vp
        _REF.ref_graph_load_edge_list.restype = vp
        _REF.ref_max_rel_err_f64.restype = f64
        _REF.ref_matmul_f32.restype = i32
        _REF.ref_matmul_f64.restype = i32
    return _REF


# ----------------------------------------------------------------------------
# Graphs
# ----------------------------------------------------------------------------
@dataclass
class HostGraph:
    """Dual index exactly as gnncg::Graph holds it (graph.hpp:34-65), split to SoA."""
    V: int
    src: np.ndarray  # edge_src[e]
    dst: np.ndarray  # edge_dst[e]
    dst_off: np.ndarray  # csr_dst.offsets
    dst_src: np.ndarray  # csr_dst.entries[].vertex
    dst_eid: np.ndarray  # csr_dst.entries[].edge
    src_off: np.ndarray  # csc_src.offsets
    src_dst: np.ndarray
    src_eid: np.ndarray

    @property
    def E(self) -> int:
        return int(self.src.shape[0])


def build_index(V: int, key: np.ndarray, other: np.ndarray):
    """Restated build_index (graph.cpp:14-28)."""
    E = key.shape[0]
    key = np.ascontiguousarray(key, dtype=np.uint32)
    other = np.ascontiguousarray(other, dtype=np.uint32)
    off = np.zeros(V + 1, np.uint64)
    nbr = np.zeros(E, np.uint32)
    eid = np.zeros(E, np.uint32)
    lib().orc_build_index(u64(V), u64(E), _p(key), _p(other), _p(off), _p(nbr), _p(eid))
    return off, nbr, eid


def host_graph(V: int, src, dst) -> HostGraph:
    """Graph from an edge list using the restated index build."""
    src = np.ascontiguousarray(src, dtype=np.uint32)
    dst = np.ascontiguousarray(dst, dtype=np.uint32)
    if src.size and (int(src.max()) >= V or int(dst.max()) >= V):
        raise ValueError("edge endpoint out of range")
    a = build_index(V, dst, src)
    b = build_index(V, src, dst)
    return HostGraph(V, src, dst, *a, *b)


class RefGraph:
    """A gnncg::Graph constructed by the reference's own code (graph.cpp:32-45)."""

    def __init__(self, handle):
        self.h = handle

    @staticmethod
    def _check(h, err):
        if not h:
            raise ValueError(err.value.decode())
        return RefGraph(h)

    @classmethod
    def from_edges(cls, V, src, dst):
        src = np.ascontiguousarray(src, dtype=np.uint32)
        dst = np.ascontiguousarray(dst, dtype=np.uint32)
        err = C.create_string_buffer(256)
        return cls._check(ref().ref_graph_new(u64(V), u64(src.size), _p(src), _p(dst), err, 256), err)

    @classmethod
    def synthetic(cls, descriptor: str, seed: int):
        err = C.create_string_buffer(256)
        return cls._check(ref().ref_graph_synthetic(descriptor.encode(), u64(seed), err, 256), err)

    @classmethod
    def load_edge_list(cls, path: str, undirected=False):
        err = C.create_string_buffer(256)
        return cls._check(ref().ref_graph_load_edge_list(path.encode(), i32(int(undirected)), err, 256), err)

    def __del__(self):
        if getattr(self, "h", None) and _REF is not None:
            _REF.ref_graph_free(vp(self.h))
            self.h = None

    def dims(self):
        V, E = u64(), u64()
        ref().ref_graph_dims(vp(self.h), C.byref(V), C.byref(E))
        return V.value, E.value

    def to_host(self) -> HostGraph:
        V, E = self.dims()
        src = np.zeros(E, np.uint32)
        dst = np.zeros(E, np.uint32)
        ref().ref_graph_edges(vp(self.h), _p(src), _p(dst))
        out = []
        for which in (0, 1):
            off = np.zeros(V + 1, np.uint64)
            nbr = np.zeros(E, np.uint32)
            eid = np.zeros(E, np.uint32)
            ref().ref_graph_index(vp(self.h), i32(which), _p(off), _p(nbr), _p(eid))
            out += [off, nbr, eid]
        return HostGraph(V, src, dst, *out)

    def degree_stats(self):
        mi, mo = u64(), u64()
        mean = f64()
        ref().ref_degree_stats(vp(self.h), C.byref(mi), C.byref(mean), C.byref(mo))
        return mi.value, mean.value, mo.value


def ref_init_seeded(rows, cols, seed, dtype=np.float64, dist=0):
    """init_seeded<T> (tensor.hpp:44-63) from the reference itself."""
    out = np.zeros((rows, cols), dtype)
    fn = ref().ref_init_seeded_f64 if dtype == np.float64 else ref().ref_init_seeded_f32
    fn(u64(rows), u64(cols), u64(seed), i32(dist), _p(out))
    return out


def ref_matmul(op: str, A: np.ndarray, B: np.ndarray):
    """op in {'nn','nt','tn'} -> matmul / matmul_nt / matmul_tn (tensor.cpp:8-60)."""
    A = np.ascontiguousarray(A)
    B = np.ascontiguousarray(B, dtype=A.dtype)
    code = {"nn": 0, "nt": 1, "tn": 2}[op]
    M = A.shape[0] if op != "tn" else A.shape[1]
    N = B.shape[1] if op != "nt" else B.shape[0]
    out = np.zeros((M, N), A.dtype)
    fn = ref().ref_matmul_f64 if A.dtype == np.float64 else ref().ref_matmul_f32
    rc = fn(i32(code), u64(A.shape[0]), u64(A.shape[1]), _p(A), u64(B.shape[0]), u64(B.shape[1]), _p(B), _p(out))
    if rc != 0:
        raise ValueError("matmul: inner dimension mismatch")
    return out


def rel_err(a, b):
    """|a-b| / max(1,|a|,|b|) elementwise (tensor.hpp:153-156)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.abs(a - b) / np.maximum(1.0, np.maximum(np.abs(a), np.abs(b)))


def max_rel_err(a, b) -> float:
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if a.shape != b.shape:
        return float("inf")
    if a.size == 0:
        return 0.0
    return float(rel_err(a, b).max())


def partition_rows(off: np.ndarray, P: int) -> np.ndarray:
    off = np.ascontiguousarray(off, dtype=np.uint64)
    bound = np.zeros(P + 1, np.uint64)
    lib().orc_partition_rows(u64(off.size - 1), _p(off), i32(P), _p(bound))
    return bound


def partition_rows_weighted(off: np.ndarray, P: int, row_weight: int) -> np.ndarray:
    """Cost-balanced row blocks (restatement of gnncg_partition_rows_weighted, include/gnncg_b200.h):
    cost(v) = off[v] + row_weight * v, bound[p] = lower_bound(cost, ceil(p * cost(V) / P)), exact
    integer arithmetic (Python ints)."""
    off = [int(x) for x in np.asarray(off, dtype=np.uint64)]
    V = len(off) - 1
    cost = [off[v] + row_weight * v for v in range(V + 1)]
    total = cost[V]
    import bisect

    bound = [0] * (P + 1)
    for p in range(1, P):
        target = -(-(p * total) // P)
        b = min(bisect.bisect_left(cost, target), V)
        bound[p] = max(b, bound[p - 1])
    bound[P] = V
    return np.array(bound, np.uint64)


# ----------------------------------------------------------------------------
# GAT
# ----------------------------------------------------------------------------
def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def gat_layer_fwd_f64(g: HostGraph, H, W, al, ar, h, f, slope=0.2):
    V = g.V
    H, W, al, ar = (_c(x, np.float64) for x in (H, W, al, ar))
    Fin = H.shape[1]
    Ht = np.zeros((V, h * f)); Al = np.zeros((V, h)); Ar = np.zeros((V, h))
    out = np.zeros((V, h * f)); m = np.zeros((V, h)); d = np.zeros((V, h))
    lib().orc_gat_layer_fwd_f64(u64(V), _p(g.dst_off), _p(g.dst_src), u64(Fin), _p(H), _p(W), _p(al), _p(ar),
                                i32(h), i32(f), f64(slope), _p(Ht), _p(Al), _p(Ar), _p(out), _p(m), _p(d))
    return dict(Ht=Ht, Al=Al, Ar=Ar, out=out, m=m, d=d)


def gat_region_fwd_f64(g: HostGraph, Ht, Al, Ar, h, f, slope=0.2):
    V = g.V
    Ht, Al, Ar = (_c(x, np.float64) for x in (Ht, Al, Ar))
    out = np.zeros((V, h * f)); m = np.zeros((V, h)); d = np.zeros((V, h))
    lib().orc_gat_region_fwd_f64(u64(V), _p(g.dst_off), _p(g.dst_src), _p(Ht), _p(Al), _p(Ar), i32(h), i32(f),
                                 f64(slope), _p(out), _p(m), _p(d))
    return dict(out=out, m=m, d=d)


def gat_region_bwd_f64(g: HostGraph, Ht, Al, Ar, al, ar, h, f, dOut, slope=0.2):
    V = g.V
    Ht, Al, Ar, al, ar, dOut = (_c(x, np.float64) for x in (Ht, Al, Ar, al, ar, dOut))
    dHt = np.zeros((V, h * f)); dAl = np.zeros((V, h)); dAr = np.zeros((V, h))
    dal = np.zeros((h, f)); dar = np.zeros((h, f))
    lib().orc_gat_region_bwd_f64(u64(V), _p(g.dst_off), _p(g.dst_src), _p(Ht), _p(Al), _p(Ar), _p(al), _p(ar),
                                 i32(h), i32(f), f64(slope), _p(dOut), _p(dHt), _p(dAl), _p(dAr), _p(dal), _p(dar))
    return dict(dHt=dHt, dAl=dAl, dAr=dAr, dal=dal, dar=dar)


def gat_layer_bwd_f64(g: HostGraph, H, W, al, ar, h, f, fwd, dOut, need_dH=True, slope=0.2):
    V = g.V
    H, W, al, ar, dOut = (_c(x, np.float64) for x in (H, W, al, ar, dOut))
    Fin = H.shape[1]
    dH = np.zeros((V, Fin)) if need_dH else None
    dW = np.zeros((Fin, h * f)); dal = np.zeros((h, f)); dar = np.zeros((h, f))
    dHt = np.zeros((V, h * f)); dAl = np.zeros((V, h)); dAr = np.zeros((V, h))
    lib().orc_gat_layer_bwd_f64(u64(V), _p(g.dst_off), _p(g.dst_src), u64(Fin), _p(H), _p(W), _p(al), _p(ar),
                                i32(h), i32(f), f64(slope), _p(fwd["Ht"]), _p(fwd["Al"]), _p(fwd["Ar"]), _p(dOut),
                                _p(dH), _p(dW), _p(dal), _p(dar), _p(dHt), _p(dAl), _p(dAr))
    return dict(dH=dH, dW=dW, dal=dal, dar=dar, dHt=dHt, dAl=dAl, dAr=dAr)


def _omp_suffix(dtype):
    dt = np.dtype(dtype)
    if dt == np.float32:
        return np.float32, "f32_omp", f32
    if dt == np.float64:
        return np.float64, "f64_omp", f64
    raise ValueError(f"unsupported dtype {dtype}")


def gat_layer_fwd_omp(g: HostGraph, H, W, al, ar, h, f, slope=0.2, dtype=np.float64):
    """The SPEC executor's forward (vertex_balanced OpenMP, stash m, d): f32 = the timed CPU
    baseline, f64 = the parity oracle at benchmark scale (oracle.cpp gat_layer_fwd_omp)."""
    dt, suf, cs = _omp_suffix(dtype)
    V = g.V
    H, W, al, ar = (_c(x, dt) for x in (H, W, al, ar))
    Fin = H.shape[1]
    z = lambda *s: np.zeros(s, dt)  # noqa: E731
    Ht, Al, Ar, out, m, d = z(V, h * f), z(V, h), z(V, h), z(V, h * f), z(V, h), z(V, h)
    getattr(lib(), "orc_gat_layer_fwd_" + suf)(u64(V), _p(g.dst_off), _p(g.dst_src), u64(Fin), _p(H), _p(W), _p(al),
                                               _p(ar), i32(h), i32(f), cs(slope), _p(Ht), _p(Al), _p(Ar), _p(out),
                                               _p(m), _p(d))
    return dict(Ht=Ht, Al=Al, Ar=Ar, out=out, m=m, d=d)


def gat_layer_bwd_omp(g: HostGraph, H, W, al, ar, h, f, fwd, dOut, need_dH=True, slope=0.2, dtype=np.float64):
    """Two-pass recompute backward (csr_dst then csc_src, no atomics) of gat_layer_fwd_omp."""
    dt, suf, cs = _omp_suffix(dtype)
    V = g.V
    H, W, al, ar, dOut = (_c(x, dt) for x in (H, W, al, ar, dOut))
    fw = {k: _c(fwd[k], dt) for k in ("Ht", "Al", "Ar", "m", "d")}
    Fin = H.shape[1]
    z = lambda *s: np.zeros(s, dt)  # noqa: E731
    dH = z(V, Fin) if need_dH else None
    dW, dal, dar = z(Fin, h * f), z(h, f), z(h, f)
    dHt, dAl, dAr, c = z(V, h * f), z(V, h), z(V, h), z(V, h)
    getattr(lib(), "orc_gat_layer_bwd_" + suf)(u64(V), _p(g.dst_off), _p(g.dst_src), _p(g.src_off), _p(g.src_dst),
                                               u64(Fin), _p(H), _p(W), _p(al), _p(ar), i32(h), i32(f), cs(slope),
                                               _p(fw["Ht"]), _p(fw["Al"]), _p(fw["Ar"]), _p(fw["m"]), _p(fw["d"]),
                                               _p(dOut), _p(dH), _p(dW), _p(dal), _p(dar), _p(dHt), _p(dAl), _p(dAr),
                                               _p(c))
    return dict(dH=dH, dW=dW, dal=dal, dar=dar, dHt=dHt, dAl=dAl, dAr=dAr, c=c)


def gat_layer_fwd_f32_omp(g: HostGraph, H, W, al, ar, h, f, slope=0.2):
    return gat_layer_fwd_omp(g, H, W, al, ar, h, f, slope, dtype=np.float32)


def gat_layer_bwd_f32_omp(g: HostGraph, H, W, al, ar, h, f, fwd, dOut, need_dH=True, slope=0.2):
    return gat_layer_bwd_omp(g, H, W, al, ar, h, f, fwd, dOut, need_dH, slope, dtype=np.float32)


# ----------------------------------------------------------------------------
# EdgeConv
# ----------------------------------------------------------------------------
NO_EDGE = 0xFFFFFFFF


def edgeconv_fwd(g: HostGraph, Th, Ph, dtype=np.float32):
    V = g.V
    Th, Ph = _c(Th, dtype), _c(Ph, dtype)
    C_ = Th.shape[1]
    out = np.zeros((V, C_), dtype)
    amax = np.zeros((V, C_), np.uint32)
    fn = lib().orc_edgeconv_fwd_f32 if dtype == np.float32 else lib().orc_edgeconv_fwd_f64
    fn(u64(V), _p(g.dst_off), _p(g.dst_src), _p(g.dst_eid), i32(C_), _p(Th), _p(Ph), _p(out), _p(amax))
    return out, amax


def edgeconv_bwd(g: HostGraph, amax, grad, dtype=np.float64):
    V = g.V
    grad = _c(grad, dtype)
    amax = _c(amax, np.uint32)
    C_ = grad.shape[1]
    dTh = np.zeros((V, C_), dtype)
    dPh = np.zeros((V, C_), dtype)
    fn = lib().orc_edgeconv_bwd_f32 if dtype == np.float32 else lib().orc_edgeconv_bwd_f64
    fn(u64(V), _p(g.dst_off), _p(g.src), i32(C_), _p(amax), _p(grad), _p(dTh), _p(dPh))
    return dTh, dPh


def edgeconv_layer_fwd_f64(g: HostGraph, H, Theta, Phi):
    V = g.V
    H, Theta, Phi = (_c(x, np.float64) for x in (H, Theta, Phi))
    Fin, C_ = Theta.shape
    Th = np.zeros((V, C_)); Ph = np.zeros((V, C_)); out = np.zeros((V, C_))
    amax = np.zeros((V, C_), np.uint32)
    lib().orc_edgeconv_layer_fwd_f64(u64(V), _p(g.dst_off), _p(g.dst_src), _p(g.dst_eid), u64(Fin), _p(H),
                                     _p(Theta), _p(Phi), i32(C_), _p(Th), _p(Ph), _p(out), _p(amax))
    return dict(Th=Th, Ph=Ph, out=out, amax=amax)


def edgeconv_layer_bwd_f64(g: HostGraph, H, Theta, Phi, amax, grad, need_dH=True):
    V = g.V
    H, Theta, Phi, grad = (_c(x, np.float64) for x in (H, Theta, Phi, grad))
    Fin, C_ = Theta.shape
    dH = np.zeros((V, Fin)) if need_dH else None
    dTheta = np.zeros((Fin, C_)); dPhi = np.zeros((Fin, C_))
    dTh = np.zeros((V, C_)); dPh = np.zeros((V, C_))
    lib().orc_edgeconv_layer_bwd_f64(u64(V), _p(g.dst_off), _p(g.src), u64(Fin), _p(H), _p(Theta), _p(Phi),
                                     i32(C_), _p(_c(amax, np.uint32)), _p(grad), _p(dH), _p(dTheta), _p(dPhi),
                                     _p(dTh), _p(dPh))
    return dict(dH=dH, dTheta=dTheta, dPhi=dPhi, dTh=dTh, dPh=dPh)


# ----------------------------------------------------------------------------
# GMMConv
# ----------------------------------------------------------------------------
def gmm_layer_fwd_f64(g: HostGraph, H, W, Pl, Pr, mu, sinv, K, r, f):
    V = g.V
    H, W, Pl, Pr, mu, sinv = (_c(x, np.float64) for x in (H, W, Pl, Pr, mu, sinv))
    Fin = H.shape[1]
    hW = np.zeros((V, K * f)); pl = np.zeros((V, r)); pr = np.zeros((V, r)); out = np.zeros((V, f))
    lib().orc_gmm_layer_fwd_f64(u64(V), _p(g.dst_off), _p(g.dst_src), u64(Fin), _p(H), _p(W), _p(Pl), _p(Pr),
                                _p(mu), _p(sinv), i32(K), i32(r), i32(f), _p(hW), _p(pl), _p(pr), _p(out))
    return dict(hW=hW, pl=pl, pr=pr, out=out)


def gmm_layer_bwd_f64(g: HostGraph, H, W, Pl, Pr, mu, sinv, K, r, f, fwd, dOut, need_dH=True):
    V = g.V
    H, W, Pl, Pr, mu, sinv, dOut = (_c(x, np.float64) for x in (H, W, Pl, Pr, mu, sinv, dOut))
    Fin = H.shape[1]
    dH = np.zeros((V, Fin)) if need_dH else None
    dW = np.zeros((Fin, K * f)); dPl = np.zeros((Fin, r)); dPr = np.zeros((Fin, r))
    dmu = np.zeros((K, r)); dsinv = np.zeros((K, r))
    dhW = np.zeros((V, K * f)); dpl = np.zeros((V, r)); dpr = np.zeros((V, r))
    lib().orc_gmm_layer_bwd_f64(u64(V), _p(g.dst_off), _p(g.dst_src), u64(Fin), _p(H), _p(W), _p(Pl), _p(Pr),
                                _p(mu), _p(sinv), i32(K), i32(r), i32(f), _p(fwd["hW"]), _p(fwd["pl"]), _p(fwd["pr"]),
                                _p(dOut), _p(dH), _p(dW), _p(dPl), _p(dPr), _p(dmu), _p(dsinv), _p(dhW), _p(dpl),
                                _p(dpr))
    return dict(dH=dH, dW=dW, dPl=dPl, dPr=dPr, dmu=dmu, dsinv=dsinv, dhW=dhW, dpl=dpl, dpr=dpr)


# ----------------------------------------------------------------------------
# GCN (PAPER.md:534-540 )
# ----------------------------------------------------------------------------
def gcn_aggregate(g: HostGraph, X, w=None, bias=None, relu=False, transpose=False, dtype=np.float64):
    """Y = act(bias + A_w X) over csr_dst (A_w^T X over csc_src when transpose)."""
    off, nbr, eid = (g.src_off, g.src_dst, g.src_eid) if transpose else (g.dst_off, g.dst_src, g.dst_eid)
    X = _c(X, dtype)
    F = X.shape[1]
    Y = np.zeros((g.V, F), dtype)
    fn = lib().orc_gcn_aggregate_f64 if dtype == np.float64 else lib().orc_gcn_aggregate_f32
    fn(u64(g.V), _p(off), _p(nbr), _p(eid), _p(None if w is None else _c(w, dtype)), i32(F), _p(X),
       _p(None if bias is None else _c(bias, dtype)), i32(int(relu)), _p(Y))
    return Y


def gcn_norm(g: HostGraph) -> np.ndarray:
    w = np.zeros(g.E, np.float32)
    lib().orc_gcn_norm(u64(g.V), u64(g.E), _p(g.src), _p(g.dst), _p(g.dst_off), _p(g.src_off), _p(w))
    return w


def gcn_layer_fwd_f64(g: HostGraph, H, W, b, w=None, relu=True):
    Ht = _c(H, np.float64) @ _c(W, np.float64)
    return dict(Ht=Ht, out=gcn_aggregate(g, Ht, w, b, relu))


def gcn_layer_bwd_f64(g: HostGraph, H, W, fwd, dOut, w=None, relu=True):
    dOut = _c(dOut, np.float64)
    dZ = np.where(fwd["out"] > 0, dOut, 0.0) if relu else dOut
    dHt = gcn_aggregate(g, dZ, w, transpose=True)
    return dict(dH=dHt @ _c(W, np.float64).T, dW=_c(H, np.float64).T @ dHt, db=dZ.sum(axis=0), dHt=dHt)


def dense_aggregate_f64(V, src, dst, H, w=None):
    src = _c(src, np.uint32); dst = _c(dst, np.uint32); H = _c(H, np.float64)
    F = H.shape[1]
    out = np.zeros((V, F))
    lib().orc_dense_aggregate_f64(u64(V), u64(src.size), _p(src), _p(dst), _p(None if w is None else _c(w, np.float64)),
                                  i32(F), _p(H), _p(out))
    return out


def cost_counts(V, E, h, f):
    L = lib()
    return dict(flops_naive=L.orc_gat_attn_flops_naive(u64(V), u64(E), u64(f)),
                flops_reorg=L.orc_gat_attn_flops_reorg(u64(V), u64(E), u64(f)),
                io_unfused=L.orc_gat_io_unfused(u64(V), u64(E), u64(h), u64(f)),
                io_fused=L.orc_gat_io_fused(u64(V), u64(E), u64(h), u64(f)))


def gen_chung_lu(V: int, E: int, offset: int, seed: int):
    """Host restatement of gnncg_gen_chung_lu (OpenMP): (src, dst) uint32, bit-identical to the
    device generator and to graph.py:chung_lu_edges_host."""
    i = np.arange(V, dtype=np.uint64)
    cdf = np.cumsum(np.uint64(1 << 40) // (i + np.uint64(offset)), dtype=np.uint64)
    src = np.zeros(E, np.uint32)
    dst = np.zeros(E, np.uint32)
    lib().orc_gen_chung_lu(u64(V), u64(E), _p(cdf), u64(seed), _p(src), _p(dst))
    return src, dst


def num_threads() -> int:
    return int(lib().orc_num_threads())
