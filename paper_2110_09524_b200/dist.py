"""Multi-GPU GAT: destination-row partitioning with one all-gather per layer (north_star).

Destination vertices are split into P contiguous row blocks of csr_dst with balanced
costs (``gnncg_partition_rows_weighted``: edges + DEFAULT_ROW_WEIGHT per row; weight 0 is the
edge-balanced ``gnncg_partition_rows``, bound[p] = lower_bound(off, ceil(p E / P))).
Rank p owns rows [r_p, r_{p+1}) and every tensor indexed by them (H, out, m, d, A_r, dOut).
Source-side tables (Ht, A_l) live in the PADDED all-gather layout: rank q's rows at
[q*maxrows, q*maxrows + n_q), so the kernels index the gathered tables directly.

A rank's in-edges are split by the owner of their source (``build_local``): local-source
edges need only the rank's own rows of Ht / A_l, remote-source edges need the all-gather.

Per layer, forward (``gnncg_gat_fwd_dist``):
  Ht, A_l, A_r = K1(H_p)            tensor-core GEMM with the LP epilogue, written straight
                                    into the rank's block of the gather tables
  all_gather(Ht || A_l)             NCCL, on the communicator's stream ...
  K2(local-source edges)            ... overlapped with the aggregation that needs no remote row
  K2(remote-source edges), merge    two online-softmax partials -> out, m, d
Backward (``gnncg_gat_bwd_dist``, fused fast mode):
  K4f(remote-source edges)          partial dHt / dA_l of other ranks' sources
  reduce_scatter(dHt || dA_l)       NCCL, overlapped with ...
  K4f(local-source edges)           ... the own sources' terms
  combine                           dHt = own + received + dA_r (x) a_r
  LP grads over the owned rows, dW_p = H_p^T dHt_p, one all-reduce of (dW, da_l, da_r)
  dH_p = dHt_p W^T
Every per-row computation touches only the rank's own rows.

The orchestration is written against a small engine interface: ``CudaEngine`` (the
product: libgnncg_b200 kernels + its NCCL communicator) here, and an oracle-backed engine in
tests/ that runs the same schedule under gloo on CPU.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from ._lib import Part, call
from .graph import DeviceIndex, DeviceSched, Workspace, _ptr, _stream, chung_lu_cdf, partition_rows
from .ops import GatParams, PROBE, gat_transform, gemm


@dataclass
class PartitionPlan:
    bounds: np.ndarray  # uint64[P+1]

    @property
    def P(self) -> int:
        return self.bounds.size - 1

    @property
    def sizes(self) -> np.ndarray:
        return np.diff(self.bounds.astype(np.int64))

    @property
    def maxrows(self) -> int:
        return int(self.sizes.max()) if self.P else 0

    @property
    def padded_V(self) -> int:
        return self.P * self.maxrows

    def owner(self, u: torch.Tensor) -> torch.Tensor:
        b = torch.as_tensor(self.bounds[1:].astype(np.int64), device=u.device)
        return torch.searchsorted(b, u, right=True)

    def padded_id(self, u: torch.Tensor) -> torch.Tensor:
        u = u.to(torch.int64)
        p = self.owner(u)
        b = torch.as_tensor(self.bounds[:-1].astype(np.int64), device=u.device)
        return p * self.maxrows + (u - b[p])

    @classmethod
    def from_dst(cls, V: int, dst: torch.Tensor, P: int, row_weight: int = 0) -> "PartitionPlan":
        deg = torch.bincount(dst.to(torch.int64), minlength=V).cpu().numpy()
        off = np.concatenate([[0], np.cumsum(deg)]).astype(np.uint64)
        return cls(partition_rows(off, P, row_weight))


@dataclass
class LocalGraph:
    """Rank-local view (gnncg_part_t): the owned destination rows' in-edges split by the owner
    of their source.  csr_*: rows = owned destinations, neighbour = padded source id;
    csc_local: rows = own sources (rebased to the block), csc_remote: rows = all padded
    sources; csc neighbours are local destination rows."""

    plan: PartitionPlan
    rank: int
    csr_local: object  # engine-specific indexes
    csr_remote: object
    csc_local: object
    csc_remote: object
    _part: object = field(default=None, repr=False)

    @property
    def num_local(self) -> int:
        return int(self.plan.sizes[self.rank])

    @property
    def row_base(self) -> int:
        return self.rank * self.plan.maxrows

    @property
    def num_edges(self) -> int:
        return int(self.csr_local.num_edges) + int(self.csr_remote.num_edges)


def build_local(plan: PartitionPlan, rank: int, src: torch.Tensor, dst: torch.Tensor, engine) -> LocalGraph:
    """Select the in-edges of the owned rows (stable in edge id), split them by source owner
    and build the four rank-local indexes."""
    r0, r1 = int(plan.bounds[rank]), int(plan.bounds[rank + 1])
    n, base, Vp = r1 - r0, rank * plan.maxrows, plan.padded_V
    d64 = dst.to(torch.int64)
    mask = (d64 >= r0) & (d64 < r1)
    ps = plan.padded_id(src.to(torch.int64)[mask])
    ld = d64[mask] - r0
    del d64, mask
    own = (ps >= base) & (ps < base + n)
    ps_l, ld_l = ps[own], ld[own]
    ps_r, ld_r = ps[~own], ld[~own]
    del ps, ld, own
    csr_local = engine.build_index(n, ld_l, ps_l, Vp)
    csc_local = engine.build_index(n, ps_l - base, ld_l, n)
    _gather_hint(csr_local, ps_l, Vp)  # K2's local pass reads Ht_all rows of the local sources
    _gather_hint(csc_local, ld_l, n)  # K4f's local pass reads dOut rows of the owned destinations
    del ps_l, ld_l
    csr_remote = engine.build_index(n, ld_r, ps_r, Vp)
    csc_remote = engine.build_index(Vp, ps_r, ld_r, n)
    _gather_hint(csr_remote, ps_r, Vp)
    _gather_hint(csc_remote, ld_r, n)
    return LocalGraph(plan, rank, csr_local, csr_remote, csc_local, csc_remote)


def _gather_hint(idx, gathered: torch.Tensor, rows: int):
    """The L2 hint of a rank-local index (gnncg_sched_t.gather_off): how often its fused kernel
    reads each row of the table it gathers, as host prefix sums (the padded Ht_all / A_l table
    for the csr passes, the owned dOut rows for the csc passes)."""
    if not hasattr(idx, "gather_off"):  # the oracle engine's indexes
        return
    cnt = torch.bincount(gathered.to(torch.int64), minlength=rows)
    off = torch.zeros(rows + 1, dtype=torch.int64, device=cnt.device)
    torch.cumsum(cnt, 0, out=off[1:])
    idx.gather_off = np.ascontiguousarray(off.cpu().numpy().view(np.uint64))


class NcclComm:
    """The library's communicator (gnncg_comm_t over NCCL) for the ranks of a torch.distributed
    group: rank 0 draws the NCCL unique id, the group broadcasts it, every rank joins."""

    def __init__(self, group=None):
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        uid = C.create_string_buffer(128)
        if self.rank == 0:
            call("gnncg_comm_unique_id", uid)
        obj = [uid.raw]
        dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
        self.handle = C.c_void_p()
        call("gnncg_comm_init", C.byref(self.handle), self.world, self.rank, C.c_char_p(obj[0]))

    def all_reduce(self, t: torch.Tensor) -> torch.Tensor:
        call("gnncg_comm_allreduce", self.handle, _ptr(t), t.numel(), _stream())
        return t

    def close(self):
        if self.handle:
            _lib.lib().gnncg_comm_destroy(self.handle)
            self.handle = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:  # interpreter shutdown
            pass


class CudaEngine:
    """The product engine: libgnncg_b200 kernels on the current CUDA device; `comm` is the
    library's NCCL communicator (None: the caller completes the gather tables and reduces the
    remote partials itself -- used to emulate ranks on one GPU)."""

    def __init__(self, device, chunk=None, comm: NcclComm | None = None):
        self.device = device
        self.ws = Workspace(device)
        self.chunk = chunk
        self.comm = comm

    def build_index(self, rows: int, key: torch.Tensor, other: torch.Tensor, n_other: int):
        from .graph import DeviceGraph

        k = key.to(torch.int32).contiguous()
        o = other.to(torch.int32).contiguous()
        return DeviceGraph.build_index(rows, k, o, self.ws, n_other)

    def _sched(self, idx: DeviceIndex) -> DeviceSched:
        return idx.sched(self.chunk) if self.chunk else idx.sched()

    def part(self, lg: LocalGraph) -> Part:
        if lg._part is None:
            idx = [lg.csr_local, lg.csr_remote, lg.csc_local, lg.csc_remote]
            keep = [(i.struct(), self._sched(i).struct()) for i in idx]
            bounds = np.ascontiguousarray(lg.plan.bounds, dtype=np.uint64)  # unpadded collectives
            pt = Part(lg.num_local, lg.plan.maxrows, lg.plan.P, lg.rank,
                      *[C.pointer(x) for pair in keep for x in pair], bounds.ctypes.data)
            lg._part = (pt, keep, bounds)
        return lg._part[0]

    def zeros(self, *shape):
        return torch.zeros(*shape, dtype=torch.float32, device=self.device)

    def empty(self, *shape):
        return torch.empty(*shape, dtype=torch.float32, device=self.device)

    def gemm(self, A, B, ta=False, tb=False, out=None):
        return gemm(A, B, trans_a=ta, trans_b=tb, out=out, ws=self.ws)

    def transform(self, H, W, a_l, a_r, p: GatParams, Ht_out, Al_out):
        """K1 with the LP epilogue on the local rows, written into the rank's block of the
        gather tables; returns A_r (destination side, local)."""
        _, _, Ar = gat_transform(H, W, a_l, a_r, p.heads, p.f, ws=self.ws, Ht=Ht_out, Al=Al_out)
        return Ar

    def _comm(self):
        return self.comm.handle if self.comm is not None else None

    def region_fwd(self, lg: LocalGraph, Ht_all, Al_all, Ar, p: GatParams):
        n = max(lg.num_local, 1)
        out, m, d = self.empty(n, p.heads * p.f), self.empty(n, p.heads), self.empty(n, p.heads)
        pt = self.part(lg)
        wp, wn = self.ws.get(_lib.lib().gnncg_gat_dist_workspace(C.byref(pt), p.heads, p.f))
        with PROBE("gat_fwd_dist"):
            call("gnncg_gat_fwd_dist", self._comm(), C.byref(pt), p.heads, p.f, p.slope, _ptr(Ht_all), _ptr(Al_all),
                 _ptr(Ar), _ptr(out), _ptr(m), _ptr(d), wp, wn, _stream())
        k = lg.num_local
        return out[:k], m[:k], d[:k]

    def region_bwd(self, lg: LocalGraph, Ht_all, Al_all, Ar, m, d, out, dOut, a_l, a_r, p: GatParams, send=None):
        """-> (dHt, dAl, dAr) of the owned rows.  `send` = (dHt_send, dAl_send) buffers to keep
        (comm None: the caller reduces them)."""
        n, h, f = max(lg.num_local, 1), p.heads, p.f
        Vp = lg.plan.padded_V
        dHt, dAl, dAr = self.empty(n, h * f), self.empty(n, h), self.empty(n, h)
        hs, als = send if send is not None else (self.empty(Vp, h * f), self.empty(Vp, h))
        pt = self.part(lg)
        wp, wn = self.ws.get(_lib.lib().gnncg_gat_dist_workspace(C.byref(pt), h, f))
        with PROBE("gat_bwd_dist"):
            call("gnncg_gat_bwd_dist", self._comm(), C.byref(pt), h, f, p.slope, _ptr(Ht_all), _ptr(Al_all), _ptr(Ar),
                 _ptr(m), _ptr(d), _ptr(out), _ptr(dOut), _ptr(a_l), _ptr(a_r), _ptr(dHt), _ptr(dAl), _ptr(dAr),
                 _ptr(hs), _ptr(als), wp, wn, _stream())
        k = lg.num_local
        return dHt[:k], dAl[:k], dAr[:k]

    def attn_grad(self, Ht, dAl, dAr, p: GatParams, out=None):
        V = Ht.shape[0]
        da_l, da_r = out if out is not None else (self.empty(p.heads, p.f), self.empty(p.heads, p.f))
        wp, wn = self.ws.get(_lib.lib().gnncg_gat_attn_grad_workspace(V, p.heads, p.f))
        with PROBE("attn_grad"):
            call("gnncg_gat_attn_grad", V, p.heads, p.f, _ptr(Ht), _ptr(dAl), _ptr(dAr), _ptr(da_l), _ptr(da_r),
                 wp, wn, _stream())
        return da_l, da_r

    def all_reduce(self, t: torch.Tensor) -> torch.Tensor:
        if self.comm is not None:
            self.comm.all_reduce(t)
        return t

    def sgd(self, param, grad, lr):
        call("gnncg_sgd_update", param.numel(), lr, _ptr(grad), _ptr(param), _stream())

    def fill_ones(self, like):
        t = torch.empty_like(like)
        call("gnncg_fill", t.numel(), 1.0, _ptr(t), _stream())
        return t

    def total(self, x, out):
        ws = torch.empty(_lib.lib().gnncg_sum_workspace(), dtype=torch.uint8, device=self.device)
        call("gnncg_sum", x.numel(), _ptr(x), _ptr(out), _ptr(ws), ws.numel(), _stream())


@dataclass
class _Layer:
    W: torch.Tensor
    a_l: torch.Tensor
    a_r: torch.Tensor
    p: GatParams


class PartitionedGAT:
    """GAT stack over a LocalGraph; identical math to models.GAT (identity between layers,
    loss = sum of exits, SGD) with the collectives of the module docstring."""

    def __init__(self, lg: LocalGraph, dims, seed=0, slope=0.2, chunk=None, engine=None, params=None):
        self.lg = lg
        if engine is None:
            dev = torch.device("cuda", torch.cuda.current_device())
            engine = CudaEngine(dev, chunk, comm=NcclComm() if dist.is_initialized() else None)
        self.engine = engine
        self.layers = []
        if params is None:
            from .models import init_uniform

            dev = self.engine.device
            gen = torch.Generator(device=dev)
            gen.manual_seed(seed)  # same seed on every rank -> identical parameters
            params = [(init_uniform(fin, h * f, gen, dev), init_uniform(h, f, gen, dev), init_uniform(h, f, gen, dev))
                      for fin, h, f in dims]
        for (W, al, ar), (fin, h, f) in zip(params, dims):
            self.layers.append(_Layer(W, al, ar, GatParams(h, f, slope)))
        self.loss = self.engine.zeros(4)

    @property
    def num_local(self):
        return self.lg.num_local

    def forward(self, H):
        E, lg = self.engine, self.lg
        Vp, b, n = lg.plan.padded_V, lg.row_base, lg.num_local
        xs, stashes = [H], []
        for L in self.layers:
            h, hf = L.p.heads, L.p.heads * L.p.f
            Ht_all, Al_all = E.empty(Vp, hf), E.empty(Vp, h)
            Ar = E.transform(xs[-1], L.W, L.a_l, L.a_r, L.p, Ht_all[b:b + n], Al_all[b:b + n])
            out, m, d = E.region_fwd(lg, Ht_all, Al_all, Ar, L.p)
            xs.append(out)
            stashes.append((Ht_all, Al_all, Ar, m, d, out))
        return xs, stashes

    def backward(self, xs, stashes, dOut):
        E, lg = self.engine, self.lg
        b, n = lg.row_base, lg.num_local
        grads = [None] * len(self.layers)
        g = dOut
        for i in reversed(range(len(self.layers))):
            L = self.layers[i]
            Ht_all, Al_all, Ar, m, d, out = stashes[i]
            dHt, dAl, dAr = E.region_bwd(lg, Ht_all, Al_all, Ar, m, d, out, g, L.a_l, L.a_r, L.p)
            # (dW, da_l, da_r) in one buffer: one all-reduce, no packing copies
            nW, hf = L.W.numel(), L.a_l.numel()
            packed = E.empty(nW + 2 * hf)
            dW, da_l, da_r = packed[:nW].view_as(L.W), packed[nW:nW + hf].view_as(L.a_l), packed[nW + hf:].view_as(L.a_r)
            E.attn_grad(Ht_all[b:b + n], dAl, dAr, L.p, out=(da_l, da_r))  # owned rows; summed by the all-reduce
            E.gemm(xs[i], dHt, ta=True, out=dW)
            E.all_reduce(packed)
            dH = E.gemm(dHt, L.W, tb=True) if i > 0 else None
            grads[i] = (dW, da_l, da_r, dH)
            g = dH
        return grads

    def train_step(self, H, lr=0.0):
        xs, stashes = self.forward(H)
        out = xs[-1]
        self.engine.total(out, self.loss)
        self.engine.all_reduce(self.loss)
        grads = self.backward(xs, stashes, self.engine.fill_ones(out))
        for L, (dW, da_l, da_r, _) in zip(self.layers, grads):
            self.engine.sgd(L.W, dW, lr)
            self.engine.sgd(L.a_l, da_l, lr)
            self.engine.sgd(L.a_r, da_r, lr)
        return self.loss[:1], grads


# Per-row work of a layer in edge units for the cost-balanced partitioner (gnncg_partition_rows_weighted):
# the slowest rank's step (per-rank emulation, scripts/emulate_ranks.py, profiles/r02_partition.txt)
# at P = 8 is lowest near 64 for both C5 (175 -> 104 ms, mean 90) and the Reddit shape (11.0 -> 8.4 ms).
DEFAULT_ROW_WEIGHT = 64


def partitioned_chung_lu(V: int, E: int, *, offset: int, seed: int, rank: int, world: int, device,
                         row_weight: int = DEFAULT_ROW_WEIGHT) -> LocalGraph:
    """This rank's share of the Chung-Lu graph gnncg_gen_chung_lu would produce, without the
    global edge list: the in-degree histogram gives the offsets the partitioner splits
    (bit-exact, gnncg_partition_rows), then gnncg_gen_chung_lu_rows regenerates the edge
    stream and keeps the rank's destination rows in edge-id order (so the local indexes
    equal the global ones restricted to the block).  Per-rank memory is O(E / P)."""
    L = _lib.lib()
    cdf = torch.from_numpy(chung_lu_cdf(V, offset).view(np.int64)).to(device)
    deg = torch.empty(V, dtype=torch.int32, device=device)
    call("gnncg_gen_chung_lu_degrees", V, E, _ptr(cdf), seed, _ptr(deg), _stream())
    off = np.zeros(V + 1, np.uint64)
    off[1:] = np.cumsum(deg.cpu().numpy().view(np.uint32), dtype=np.uint64)
    del deg
    plan = PartitionPlan(partition_rows(off, world, row_weight))
    r0, r1 = int(plan.bounds[rank]), int(plan.bounds[rank + 1])
    n = int(off[r1] - off[r0])
    src = torch.empty(max(n, 1), dtype=torch.int32, device=device)
    dst = torch.empty(max(n, 1), dtype=torch.int32, device=device)
    ws = torch.empty(L.gnncg_gen_chung_lu_rows_workspace(E), dtype=torch.uint8, device=device)
    call("gnncg_gen_chung_lu_rows", V, E, _ptr(cdf), seed, r0, r1, _ptr(src), _ptr(dst), _ptr(ws), ws.numel(),
         _stream())
    del ws, cdf
    engine = CudaEngine(device)
    return build_local(plan, rank, src[:n], dst[:n], engine)
