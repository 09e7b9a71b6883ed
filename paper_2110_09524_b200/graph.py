"""Device-resident graph store: the B200 counterpart of gnncg::Graph (graph.hpp:34-65).

A :class:`DeviceGraph` holds both indexes of the reference's dual-index graph in
HBM as structure-of-arrays:

  csr_dst  -- in-edges grouped by destination  (Graph::csr_dst, graph.hpp:44)
  csc_src  -- out-edges grouped by source      (Graph::csc_src, graph.hpp:46)
  edge_src / edge_dst -- the input edge list   (graph.hpp:48-49)

Both indexes are built ON THE DEVICE by ``gnncg_csr_build`` and are
bit-identical to the reference's ``build_index`` (graph.cpp:14-28).  Schedules
(edge-balance work items, see gnncg_sched_t) are derived once per index and
cached.

Host-side generators reproduce the reference's descriptor idea
(``generate_synthetic``, graph.cpp:157-249) for the benchmark shapes the reference
cannot produce at scale: exact-E uniform graphs (Cora / Pubmed shaped),
Chung-Lu power-law graphs (Reddit shaped, generated on the device), and kNN
point-cloud graphs (ModelNet40 shaped).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._lib import Index, Sched, call, i64, u64

DEFAULT_CHUNK = 2048  # max edges per work item before a row is split (edge balance)


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _stream(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


@dataclass
class DeviceIndex:
    """One AdjIndex in HBM: off (int64 holding u64), nbr / eid (int32 holding u32)."""

    off: torch.Tensor
    nbr: torch.Tensor
    eid: torch.Tensor | None
    _struct: Index | None = field(default=None, repr=False)
    _sched: dict = field(default_factory=dict, repr=False)
    # host uint64 offsets of the other index of the same graph: how often the fused kernel over
    # THIS index reads each row of the table it gathers (gnncg_sched_t.gather_off, L2 hint)
    gather_off: np.ndarray | None = field(default=None, repr=False)

    @property
    def num_rows(self) -> int:
        return self.off.numel() - 1

    @property
    def num_edges(self) -> int:
        return self.nbr.numel()

    def struct(self) -> Index:
        if self._struct is None:
            self._struct = Index(self.num_rows, self.num_edges, _ptr(self.off), _ptr(self.nbr), _ptr(self.eid))
        return self._struct

    def sched(self, chunk: int = DEFAULT_CHUNK) -> "DeviceSched":
        if chunk not in self._sched:
            sc = DeviceSched.build(self.off.cpu().numpy().view(np.uint64), chunk, self.off.device)
            sc.gather_off = self.gather_off
            self._sched[chunk] = sc
        return self._sched[chunk]

    def max_degree(self) -> int:
        out = u64()
        call("gnncg_max_degree", C.byref(self.struct()), C.byref(out), _stream())
        return int(out.value)

    def to_host(self):
        """(off, nbr, eid) as numpy uint64 / uint32 arrays."""
        off = self.off.cpu().numpy().view(np.uint64)
        nbr = self.nbr.cpu().numpy().view(np.uint32)
        eid = None if self.eid is None else self.eid.cpu().numpy().view(np.uint32)
        return off, nbr, eid


@dataclass
class DeviceSched:
    """gnncg_sched_t in HBM.  Work items: split-row chunks first, then whole rows."""

    num_items: int
    num_split_items: int
    num_split_rows: int
    chunk: int
    items: torch.Tensor
    split_rows: torch.Tensor
    split_first: torch.Tensor
    gather_off: np.ndarray | None = None
    _struct: Sched | None = field(default=None, repr=False)

    @staticmethod
    def host_arrays(off: np.ndarray, chunk: int):
        off = np.ascontiguousarray(off, dtype=np.uint64)
        rows = off.size - 1
        n, ns, nr = i64(), i64(), i64()
        L = _lib.lib()
        _lib.check(L.gnncg_sched_build_host(rows, off.ctypes.data, chunk, C.byref(n), C.byref(ns), C.byref(nr),
                                            None, None, None), "gnncg_sched_build_host")
        items = np.zeros(2 * max(n.value, 1), np.uint32)
        split_rows = np.zeros(max(nr.value, 1), np.uint32)
        split_first = np.zeros(nr.value + 1, np.uint32)
        _lib.check(L.gnncg_sched_build_host(rows, off.ctypes.data, chunk, C.byref(n), C.byref(ns), C.byref(nr),
                                            items.ctypes.data, split_rows.ctypes.data, split_first.ctypes.data),
                   "gnncg_sched_build_host")
        return n.value, ns.value, nr.value, items, split_rows, split_first

    @classmethod
    def build(cls, off: np.ndarray, chunk: int, device) -> "DeviceSched":
        n, ns, nr, items, split_rows, split_first = cls.host_arrays(off, chunk)
        up = lambda a: torch.from_numpy(a.view(np.int32)).to(device)  # noqa: E731
        return cls(n, ns, nr, chunk, up(items), up(split_rows), up(split_first))

    def struct(self) -> Sched:
        if self._struct is None:
            go = self.gather_off
            self._struct = Sched(self.num_items, self.num_split_items, self.num_split_rows, self.chunk, 0,
                                 _ptr(self.items), _ptr(self.split_rows), _ptr(self.split_first),
                                 None if go is None else go.ctypes.data, 0 if go is None else go.size - 1)
        return self._struct


class Workspace:
    """Grow-only device scratch shared by the calls of one graph (never allocated in a hot call
    once warm).  The GAT calls keep per-call state in it (split-row partials and the work
    counter of the item fetch), so calls that may run concurrently -- on different streams --
    need one Workspace each; calls on one stream can share it."""

    def __init__(self, device):
        self.device = device
        self.buf = torch.empty(0, dtype=torch.uint8, device=device)

    def get(self, nbytes: int) -> tuple[int, int]:
        if nbytes > self.buf.numel():
            self.buf = torch.empty(int(nbytes * 1.25) + 256, dtype=torch.uint8, device=self.device)
        return (self.buf.data_ptr() if self.buf.numel() else None), self.buf.numel()


class DeviceGraph:
    """Immutable dual-index graph in HBM (gnncg::Graph, graph.hpp:34-65)."""

    def __init__(self, num_vertices: int, edge_src: torch.Tensor, edge_dst: torch.Tensor, csr_dst: DeviceIndex,
                 csc_src: DeviceIndex):
        self.num_vertices = int(num_vertices)
        self.edge_src = edge_src
        self.edge_dst = edge_dst
        self.csr_dst = csr_dst
        self.csc_src = csc_src
        self.device = edge_src.device
        self.ws = Workspace(self.device)

    @property
    def num_edges(self) -> int:
        return self.edge_src.numel()

    # -- construction ------------------------------------------------------
    @staticmethod
    def build_index(V: int, key: torch.Tensor, other: torch.Tensor, ws: Workspace, n_other: int | None = None
                    ) -> DeviceIndex:
        """Device counting sort by key vertex, stable in edge id (graph.cpp:14-28).  Keys range
        over [0, V), neighbour ids over [0, n_other) (default V; larger for rank-local indexes)."""
        E = key.numel()
        dev = key.device
        off = torch.empty(V + 1, dtype=torch.int64, device=dev)
        nbr = torch.empty(E, dtype=torch.int32, device=dev)
        eid = torch.empty(E, dtype=torch.int32, device=dev)
        need = _lib.lib().gnncg_csr_build_workspace(V, E)
        wp, wn = ws.get(need)
        call("gnncg_csr_build_rect", V, V if n_other is None else n_other, E, _ptr(key), _ptr(other), _ptr(off),
             _ptr(nbr), _ptr(eid), wp, wn, _stream())
        return DeviceIndex(off, nbr, eid)

    @classmethod
    def from_device_edges(cls, V: int, src: torch.Tensor, dst: torch.Tensor) -> "DeviceGraph":
        """Graph(V, edges) (graph.cpp:32-45): edge i = (src[i], dst[i]).  Raises GraphError on
        an out-of-range endpoint, like the reference."""
        _lib.require_device()
        src = src.to(torch.int32).contiguous()
        dst = dst.to(torch.int32).contiguous()
        ws = Workspace(src.device)
        csr = cls.build_index(V, dst, src, ws)
        csc = cls.build_index(V, src, dst, ws)
        # L2 hint: K2 over csr_dst gathers source rows (read out-degree times), K4f over csc_src
        # gathers destination rows (read in-degree times)
        csr.gather_off = np.ascontiguousarray(csc.off.cpu().numpy().view(np.uint64))
        csc.gather_off = np.ascontiguousarray(csr.off.cpu().numpy().view(np.uint64))
        g = cls(V, src, dst, csr, csc)
        g.ws = ws
        return g

    @classmethod
    def from_edges(cls, V: int, src, dst, device="cuda") -> "DeviceGraph":
        """From a host edge list (numpy / sequences of non-negative ints)."""
        s = np.ascontiguousarray(np.asarray(src, dtype=np.int64))
        d = np.ascontiguousarray(np.asarray(dst, dtype=np.int64))
        if s.shape != d.shape:
            raise _lib.TensorError("from_edges: src/dst length mismatch")
        if s.size and (s.min() < 0 or d.min() < 0 or s.max() >= 2**32 or d.max() >= 2**32):
            raise _lib.GraphError("edge endpoint out of range")
        ts = torch.from_numpy(s.astype(np.uint32).view(np.int32)).to(device)
        td = torch.from_numpy(d.astype(np.uint32).view(np.int32)).to(device)
        return cls.from_device_edges(V, ts, td)

    @classmethod
    def chung_lu(cls, V: int, E: int, *, offset: int = 1100, seed: int = 0, device="cuda") -> "DeviceGraph":
        """Reddit-shaped power-law graph: Chung-Lu with integer weights w_i = floor(2^40 / (i + offset))
        for both endpoints (Zipf, gamma = 2, degree cap ~ E / (offset ln(V/offset+1))).  Generated on
        the device from a counter-based hash, so (V, E, offset, seed) fixes the edge list exactly."""
        _lib.require_device()
        cdf = chung_lu_cdf(V, offset)
        tcdf = torch.from_numpy(cdf.view(np.int64)).to(device)
        src = torch.empty(E, dtype=torch.int32, device=device)
        dst = torch.empty(E, dtype=torch.int32, device=device)
        call("gnncg_gen_chung_lu", V, E, _ptr(tcdf), seed, _ptr(src), _ptr(dst), _stream())
        return cls.from_device_edges(V, src, dst)

    # -- relabeling ---------------------------------------------------------
    def degree_order(self) -> torch.Tensor:
        """perm (int64, device): perm[new] = old id, vertices by descending in + out degree (ties:
        lower old id first).  Relabeling with it puts the rows the fused kernels gather most often
        at the low ids, where the L2-persisting window (gnncg_l2_persist) can cover them for any
        input labelling.  Preprocessing on torch, outside any training step."""
        deg = (self.csr_dst.off[1:] - self.csr_dst.off[:-1]) + (self.csc_src.off[1:] - self.csc_src.off[:-1])
        return torch.sort(-deg, stable=True).indices

    def relabel(self, perm: torch.Tensor) -> "DeviceGraph":
        """The same graph with vertex old = perm[new] renamed new (edge ids unchanged: edge i is
        still edge i, so per-row edge order, EdgeConv argmax ids and results are unchanged up to
        the renaming).  Inputs follow with permute_rows(X, perm); outputs map back with
        unpermute_rows(Y, perm)."""
        V = self.num_vertices
        perm = perm.to(device=self.device, dtype=torch.int64)
        if perm.numel() != V:
            raise _lib.TensorError("relabel: perm must have num_vertices entries")
        inv = torch.empty_like(perm)
        inv[perm] = torch.arange(V, device=self.device)
        src = inv[self.edge_src.to(torch.int64) & 0xFFFFFFFF].to(torch.int32)
        dst = inv[self.edge_dst.to(torch.int64) & 0xFFFFFFFF].to(torch.int32)
        return DeviceGraph.from_device_edges(V, src, dst)

    # -- queries -----------------------------------------------------------
    def index(self, which: str) -> DeviceIndex:
        return self.csr_dst if which == "dst" else self.csc_src

    def degree_stats(self):
        """degree_stats (graph.cpp:47-57): (max_in, mean_in, max_out)."""
        V = self.num_vertices
        mean = 0.0 if V == 0 else float(self.num_edges) / float(V)
        return self.csr_dst.max_degree(), mean, self.csc_src.max_degree()

    def to_host(self):
        """Everything a gnncg::Graph holds, as numpy arrays (for parity checks)."""
        d = self.csr_dst.to_host()
        s = self.csc_src.to_host()
        return dict(V=self.num_vertices, src=self.edge_src.cpu().numpy().view(np.uint32),
                    dst=self.edge_dst.cpu().numpy().view(np.uint32), dst_off=d[0], dst_src=d[1], dst_eid=d[2],
                    src_off=s[0], src_dst=s[1], src_eid=s[2])


def permute_rows(X: torch.Tensor, perm: torch.Tensor) -> torch.Tensor:
    """Rows of X in the relabeled order: out[new] = X[perm[new]] (DeviceGraph.relabel)."""
    return X.index_select(0, perm.to(device=X.device, dtype=torch.int64))


def unpermute_rows(Y: torch.Tensor, perm: torch.Tensor) -> torch.Tensor:
    """Rows of a relabeled result back in the original order: out[perm[new]] = Y[new]."""
    out = torch.empty_like(Y)
    out.index_copy_(0, perm.to(device=Y.device, dtype=torch.int64), Y)
    return out


# ---------------------------------------------------------------------------
# Host-side generators (deterministic for a fixed seed)
# ---------------------------------------------------------------------------
def chung_lu_cdf(V: int, offset: int) -> np.ndarray:
    """Inclusive prefix sums of w_i = floor(2^40 / (i + offset)) (exact integer arithmetic)."""
    i = np.arange(V, dtype=np.uint64)
    w = np.uint64(1 << 40) // (i + np.uint64(offset))
    return np.cumsum(w, dtype=np.uint64)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """Host restatement of the device hash (graph.cu:splitmix64), numpy uint64 wrap-around."""
    with np.errstate(over="ignore"):
        x = x + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return x ^ (x >> np.uint64(31))


def mulhi64(a: np.ndarray, b: int) -> np.ndarray:
    """High 64 bits of the 128-bit product a*b (== __umul64hi), vectorised in uint64."""
    m32 = np.uint64(0xFFFFFFFF)
    s32 = np.uint64(32)
    b = np.uint64(b)
    a_lo, a_hi = a & m32, a >> s32
    b_lo, b_hi = b & m32, b >> s32
    ll, lh, hl, hh = a_lo * b_lo, a_lo * b_hi, a_hi * b_lo, a_hi * b_hi
    mid = (ll >> s32) + (lh & m32) + (hl & m32)
    return hh + (lh >> s32) + (hl >> s32) + (mid >> s32)


def chung_lu_edges_host(V: int, E: int, offset: int, seed: int):
    """Host restatement of gnncg_gen_chung_lu: returns (src, dst) bit-identical to the device."""
    cdf = chung_lu_cdf(V, offset)
    total = int(cdf[-1])
    out = []
    for lo in range(0, E, 1 << 24):
        e = np.arange(lo, min(E, lo + (1 << 24)), dtype=np.uint64)
        with np.errstate(over="ignore"):
            base = np.uint64(seed) * np.uint64(0xD1B54A32D192ED03) + np.uint64(2) * e
            h0 = splitmix64(base)
            h1 = splitmix64(base + np.uint64(1))
            s = np.searchsorted(cdf, mulhi64(h1, total), side="right").astype(np.uint32)
            d = np.searchsorted(cdf, mulhi64(h0, total), side="right").astype(np.uint32)
        out.append((s, d))
    if not out:
        return np.zeros(0, np.uint32), np.zeros(0, np.uint32)
    return np.concatenate([o[0] for o in out]), np.concatenate([o[1] for o in out])


def uniform_edges(V: int, E: int, seed: int):
    """Exact-E uniform random directed edges (Cora / Pubmed shaped), self-loops kept."""
    rng = np.random.default_rng(seed)
    src = rng.integers(0, V, E, dtype=np.int64).astype(np.uint32)
    dst = rng.integers(0, V, E, dtype=np.int64).astype(np.uint32)
    return src, dst


def knn_edges(clouds: int, points: int, k: int, seed: int):
    """ModelNet40-shaped batch: `clouds` clouds of `points` points uniform in [-1,1]^3.
    Edges u -> v for the k nearest neighbours u of every point v (self excluded, ties by lower
    index), listed v-major in ascending (distance, index) order; vertex id = cloud*points + i."""
    rng = np.random.default_rng(seed)
    src_all, dst_all = [], []
    for c in range(clouds):
        x = rng.uniform(-1.0, 1.0, (points, 3))
        d2 = ((x[:, None, :] - x[None, :, :]) ** 2).sum(-1)
        np.fill_diagonal(d2, np.inf)
        nn = np.argsort(d2, axis=1, kind="stable")[:, :k]  # stable: lower index first on ties
        base = c * points
        dst_all.append(np.repeat(np.arange(points), k) + base)
        src_all.append(nn.reshape(-1) + base)
    return (np.concatenate(src_all).astype(np.uint32), np.concatenate(dst_all).astype(np.uint32))


def partition_rows(off: np.ndarray, parts: int, row_weight: int = 0) -> np.ndarray:
    """Row-block partitioner: bound[p] = lower_bound(off, ceil(p*E/P)) (bit-exact, host); with
    row_weight > 0 the cost-balanced variant, cost(v) = off[v] + row_weight * v."""
    off = np.ascontiguousarray(off, dtype=np.uint64)
    bound = np.zeros(parts + 1, np.uint64)
    if row_weight:
        call("gnncg_partition_rows_weighted", off.size - 1, off.ctypes.data, parts, int(row_weight), bound.ctypes.data)
    else:
        call("gnncg_partition_rows", off.size - 1, off.ctypes.data, parts, bound.ctypes.data)
    return bound
