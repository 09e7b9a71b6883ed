"""Multi-GPU GAT: destination-row partitioning with one all-gather per layer (north_star).

Destination vertices are split into P contiguous row blocks of csr_dst with balanced
edge counts (``gnncg_partition_rows``: bound[p] = lower_bound(off, ceil(p E / P))).
Rank p owns rows [r_p, r_{p+1}) and every tensor indexed by them (H, out, m, d, A_r, dOut).

Per layer, forward:
  Ht_p, A_l,p, A_r,p = K1(H_p)      (one tensor-core GEMM with the LP epilogue, local rows)
  all_gather(Ht), all_gather(A_l)   (NCCL over NVLink; blocks padded to the largest)
  K2 over the local csr_dst block   (no collective: destination rows are independent)
Backward:
  K3 over the local csr_dst block   (c, dA_r: local)
  K4 over the local csc_src         (rows = all sources, neighbours = local rows):
                                    partial dHt / dA_l for every source
  reduce_scatter(dHt), reduce_scatter(dA_l) -> the owned rows (the terms are linear)
  LP grads over the owned rows, dW_p = H_p^T dHt_p -> all_reduce (tiny)
  dH_p = dHt_p W^T
Every per-row computation touches only the rank's own rows; the gathered tensors are read
only by the fused kernels.

Source ids inside the local indexes are remapped to the PADDED global layout of the
all-gather buffer (block p at rows [p*maxrows, p*maxrows + n_p)), so the kernels index
the gathered tensors directly.  The orchestration is written against a small engine
interface: ``CudaEngine`` (the product: libgnncg_b200 + NCCL) here, and an oracle-backed
engine in tests/ that runs the same schedule under gloo on CPU.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from ._lib import call
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
    def from_dst(cls, V: int, dst: torch.Tensor, P: int) -> "PartitionPlan":
        deg = torch.bincount(dst.to(torch.int64), minlength=V).cpu().numpy()
        off = np.concatenate([[0], np.cumsum(deg)]).astype(np.uint64)
        return cls(partition_rows(off, P))


@dataclass
class LocalGraph:
    """Rank-local view: csr over owned destination rows, csc over all (padded) sources."""

    plan: PartitionPlan
    rank: int
    csr: object  # engine-specific index
    csc: object

    @property
    def num_local(self) -> int:
        return int(self.plan.sizes[self.rank])

    @property
    def row_base(self) -> int:
        return self.rank * self.plan.maxrows


def build_local(plan: PartitionPlan, rank: int, src: torch.Tensor, dst: torch.Tensor, engine) -> LocalGraph:
    """Select the in-edges of the owned rows (stable in edge id) and build both local indexes."""
    r0, r1 = int(plan.bounds[rank]), int(plan.bounds[rank + 1])
    d64 = dst.to(torch.int64)
    mask = (d64 >= r0) & (d64 < r1)
    ls = plan.padded_id(src.to(torch.int64)[mask])
    ld = d64[mask] - r0
    csr = engine.build_index(r1 - r0, ld, ls, plan.padded_V)
    csc = engine.build_index(plan.padded_V, ls, ld, r1 - r0)
    return LocalGraph(plan, rank, csr, csc)


class CudaEngine:
    """The product engine: libgnncg_b200 kernels on the current CUDA device."""

    def __init__(self, device, chunk=None, mode="auto"):
        self.device = device
        self.ws = Workspace(device)
        self.chunk = chunk
        self.mode = mode

    def build_index(self, rows: int, key: torch.Tensor, other: torch.Tensor, n_other: int):
        from .graph import DeviceGraph

        k = key.to(torch.int32).contiguous()
        o = other.to(torch.int32).contiguous()
        return DeviceGraph.build_index(rows, k, o, self.ws, n_other)

    def _sched(self, idx: DeviceIndex) -> DeviceSched:
        return idx.sched(self.chunk) if self.chunk else idx.sched()

    def zeros(self, *shape):
        return torch.zeros(*shape, dtype=torch.float32, device=self.device)

    def empty(self, *shape):
        return torch.empty(*shape, dtype=torch.float32, device=self.device)

    def gemm(self, A, B, ta=False, tb=False):
        return gemm(A, B, trans_a=ta, trans_b=tb, ws=self.ws)

    def transform(self, H, W, a_l, a_r, p: GatParams):
        """K1 with the LP epilogue on the local rows: (Ht, A_l, A_r)."""
        return gat_transform(H, W, a_l, a_r, p.heads, p.f, ws=self.ws)

    def attn_dots(self, Ht, a_l, a_r, p: GatParams):
        V = Ht.shape[0]
        Al, Ar = self.empty(V, p.heads), self.empty(V, p.heads)
        with PROBE("attn_dots"):
            call("gnncg_gat_attn_dots", V, p.heads, p.f, _ptr(Ht), _ptr(a_l), _ptr(a_r), _ptr(Al), _ptr(Ar),
                 _stream())
        return Al, Ar

    def region_fwd(self, lg: LocalGraph, Ht, Al, Ar_local, p: GatParams):
        n = lg.num_local
        out, m, d = self.empty(n, p.heads * p.f), self.empty(n, p.heads), self.empty(n, p.heads)
        s = self._sched(lg.csr)
        wp, wn = self.ws.get(_lib.lib().gnncg_gat_workspace(s.struct(), None, p.heads, p.f))
        with PROBE("gat_fwd"):
            call("gnncg_gat_fwd", lg.csr.struct(), s.struct(), p.heads, p.f, p.slope, _ptr(Ht), _ptr(Al),
                 _ptr(Ar_local), _ptr(out), _ptr(m), _ptr(d), wp, wn, _stream())
        return out, m, d

    def region_bwd(self, lg: LocalGraph, Ht, Al, Ar_local, m, d, dOut, a_l, a_r, p: GatParams, out=None):
        """K3 + K4 (or the fused fast pass) -> (dHt partial over padded sources, dAl partial, dAr local)."""
        n, h, f = lg.num_local, p.heads, p.f
        c, dAr = self.empty(n, h), self.empty(n, h)
        sd, ss = self._sched(lg.csr), self._sched(lg.csc)
        Vp = lg.plan.padded_V
        dHt, dAl = self.empty(Vp, h * f), self.empty(Vp, h)
        wp, wn = self.ws.get(_lib.lib().gnncg_gat_workspace(sd.struct(), ss.struct(), h, f))
        st = _stream()
        if out is not None and self.mode != "deterministic" and _lib.lib().gnncg_gat_fast_supported(h, f):
            rec = self.empty(n, _lib.lib().gnncg_gat_rec_stride(h))
            Ar_loc = Ar_local.contiguous()
            with PROBE("gat_bwd_prep"):
                call("gnncg_gat_bwd_prep", n, h, f, _ptr(dOut), _ptr(out), _ptr(Ar_loc), _ptr(m), _ptr(d), _ptr(rec),
                     st)
            with PROBE("gat_bwd_src_fused"):
                call("gnncg_gat_bwd_src_fused", lg.csc.struct(), ss.struct(), h, f, p.slope, lg.row_base, n,
                     _ptr(Ht), _ptr(Al), _ptr(rec), _ptr(dOut), _ptr(a_l), _ptr(a_r), _ptr(dHt), _ptr(dAl), _ptr(dAr),
                     wp, wn, st)
            return dHt, dAl, dAr
        with PROBE("gat_bwd_dst"):
            call("gnncg_gat_bwd_dst", lg.csr.struct(), sd.struct(), h, f, p.slope, _ptr(Ht), _ptr(Al),
                 _ptr(Ar_local), _ptr(m), _ptr(d), _ptr(dOut), _ptr(c), _ptr(dAr), wp, wn, st)
        with PROBE("gat_bwd_src"):
            call("gnncg_gat_bwd_src", lg.csc.struct(), ss.struct(), h, f, p.slope, lg.row_base, n, _ptr(Ht),
                 _ptr(Al), _ptr(Ar_local), _ptr(m), _ptr(d), _ptr(c), _ptr(dOut), _ptr(dAr), _ptr(a_l), _ptr(a_r),
                 _ptr(dHt), _ptr(dAl), wp, wn, st)
        return dHt, dAl, dAr

    def attn_grad(self, Ht, dAl, dAr, p: GatParams):
        V = Ht.shape[0]
        da_l, da_r = self.empty(p.heads, p.f), self.empty(p.heads, p.f)
        wp, wn = self.ws.get(_lib.lib().gnncg_gat_attn_grad_workspace(V, p.heads, p.f))
        with PROBE("attn_grad"):
            call("gnncg_gat_attn_grad", V, p.heads, p.f, _ptr(Ht), _ptr(dAl), _ptr(dAr), _ptr(da_l), _ptr(da_r),
                 wp, wn, _stream())
        return da_l, da_r

    def sgd(self, param, grad, lr):
        call("gnncg_sgd_update", param.numel(), lr, _ptr(grad), _ptr(param), _stream())

    def fill_ones(self, like):
        t = torch.empty_like(like)
        call("gnncg_fill", t.numel(), 1.0, _ptr(t), _stream())
        return t

    def total(self, x, out):
        ws = torch.empty(_lib.lib().gnncg_sum_workspace(), dtype=torch.uint8, device=self.device)
        call("gnncg_sum", x.numel(), _ptr(x), _ptr(out), _ptr(ws), ws.numel(), _stream())


class Comm:
    """torch.distributed collectives over the padded row-block layout."""

    def __init__(self, group=None):
        self.group = group

    def all_gather_rows(self, local: torch.Tensor, maxrows: int) -> torch.Tensor:
        P = dist.get_world_size(self.group)
        n, cols = local.shape
        if n == maxrows:
            send = local.contiguous()
        else:
            send = torch.zeros(maxrows, cols, dtype=local.dtype, device=local.device)
            send[:n] = local
        out = torch.empty(P * maxrows, cols, dtype=local.dtype, device=local.device)
        dist.all_gather_into_tensor(out, send, group=self.group)
        return out

    def reduce_scatter_rows(self, full: torch.Tensor, maxrows: int, n: int) -> torch.Tensor:
        out = torch.empty(maxrows, full.shape[1], dtype=full.dtype, device=full.device)
        dist.reduce_scatter_tensor(out, full.contiguous(), op=dist.ReduceOp.SUM, group=self.group)
        return out[:n]

    def all_reduce(self, t: torch.Tensor) -> torch.Tensor:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return t


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
        self.engine = engine or CudaEngine(torch.device("cuda", torch.cuda.current_device()), chunk)
        self.comm = Comm()
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
        E, lg, mr = self.engine, self.lg, self.lg.plan.maxrows
        xs, stashes = [H], []
        for L in self.layers:
            Ht_local, Al_local, Ar_local = E.transform(xs[-1], L.W, L.a_l, L.a_r, L.p)
            Ht = self.comm.all_gather_rows(Ht_local, mr)
            Al = self.comm.all_gather_rows(Al_local, mr)
            out, m, d = E.region_fwd(lg, Ht, Al, Ar_local, L.p)
            xs.append(out)
            stashes.append((Ht, Ht_local, Al, Ar_local, m, d, out))
        return xs, stashes

    def backward(self, xs, stashes, dOut):
        E, lg = self.engine, self.lg
        mr, n = lg.plan.maxrows, lg.num_local
        grads = [None] * len(self.layers)
        g = dOut
        for i in reversed(range(len(self.layers))):
            L = self.layers[i]
            Ht, Ht_local, Al, Ar_local, m, d, out = stashes[i]
            dHt_part, dAl_part, dAr = E.region_bwd(lg, Ht, Al, Ar_local, m, d, g, L.a_l, L.a_r, L.p, out=out)
            dHt = self.comm.reduce_scatter_rows(dHt_part, mr, n)
            dAl = self.comm.reduce_scatter_rows(dAl_part, mr, n)
            da_l, da_r = E.attn_grad(Ht_local, dAl, dAr, L.p)  # owned rows only; summed by the all-reduce
            dW = E.gemm(xs[i], dHt, ta=True)
            packed = torch.cat([dW.reshape(-1), da_l.reshape(-1), da_r.reshape(-1)])
            self.comm.all_reduce(packed)
            nW = dW.numel()
            dW = packed[:nW].view_as(dW)
            da_l = packed[nW:nW + da_l.numel()].view_as(da_l)
            da_r = packed[nW + da_l.numel():].view_as(da_r)
            dH = E.gemm(dHt, L.W, tb=True) if i > 0 else None
            grads[i] = (dW, da_l, da_r, dH)
            g = dH
        return grads

    def train_step(self, H, lr=0.0):
        xs, stashes = self.forward(H)
        out = xs[-1]
        self.engine.total(out, self.loss)
        self.comm.all_reduce(self.loss)
        grads = self.backward(xs, stashes, self.engine.fill_ones(out))
        for L, (dW, da_l, da_r, _) in zip(self.layers, grads):
            self.engine.sgd(L.W, dW, lr)
            self.engine.sgd(L.a_l, da_l, lr)
            self.engine.sgd(L.a_r, da_r, lr)
        return self.loss[:1], grads


def partitioned_chung_lu(V: int, E: int, *, offset: int, seed: int, rank: int, world: int, device) -> LocalGraph:
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
    plan = PartitionPlan(partition_rows(off, world))
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
