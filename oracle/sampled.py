"""TEST INFRASTRUCTURE ONLY -- f64 restatement of one GAT layer on SAMPLED rows.

The full-graph oracle (oracle.cpp) needs the whole graph in host memory and minutes of CPU
time at the benchmark sizes (C2: 114M edges; C5: 1B edges).  A GAT layer's value at one row
depends only on a bounded neighbourhood, so sampled rows can be checked exactly in f64 from
the local neighbourhood of each row:

  forward, destination v   (edge-softmax RS1/RS2 PAPER.md:527-530):
      Ht = H W ; A_l = <Ht, a_l>_k ; A_r = <Ht, a_r>_k ; s_e = LReLU(A_l[u] + A_r[v])
      out[v] = sum_{e=(u->v)} softmax_v(s)_e Ht[u]          needs Ht on in(v) + {v}
  backward, source u       (App. B; loss seed SPEC.md:217):
      alpha_uv, dalpha_uv = <dOut[v], Ht[u]>_k, c[v] = sum_{u' in in(v)} alpha dalpha
      dz_uv = LReLU'(z) alpha (dalpha - c[v])
      dHt[u] = sum_{v in out(u)} alpha_uv dOut[v] + dA_l[u] (x) a_l + dA_r[u] (x) a_r
      dA_l[u] = sum_{v in out(u)} dz_uv ;  dA_r[u] = sum_{u' in in(u)} dz_u'u
      dH[u] = dHt[u] W^T                                    needs Ht on in(out(u)), in(u)
Empty in-neighbourhood: out = 0.  Comparator: rel_err (tensor.hpp:153-156).

Only tests/, __graft_entry__.smoke() and bench.py's checker leg import this module; it is
never the thing measured.  `src` is any object with
    in_nbrs(v) -> np.ndarray of source ids of v's in-edges (csr_dst row, edge-id order)
    out_nbrs(u) -> np.ndarray of destination ids of u's out-edges (csc_src row)
    rows(ids) -> np.ndarray [len(ids), F_in] of the layer input H (any float dtype)
    dout(ids) -> np.ndarray [len(ids), h*f] of the layer's output gradient (backward only)
"""
from __future__ import annotations

import numpy as np


def _lrelu(z, slope):
    return np.where(z > 0, z, slope * z)


class _Tables:
    """Ht / A_l / A_r in f64 on a set of rows of the layer input (sorted ids)."""

    def __init__(self, src, W, a_l, a_r, h, f):
        self.src, self.h, self.f = src, h, f
        self.W = np.asarray(W, np.float64)
        self.a_l = np.asarray(a_l, np.float64).reshape(h, f)
        self.a_r = np.asarray(a_r, np.float64).reshape(h, f)
        self.ids = np.zeros(0, np.int64)
        self.Ht = np.zeros((0, h * f))

    def need(self, ids):
        new = np.setdiff1d(np.unique(np.asarray(ids, np.int64)), self.ids)
        if new.size:
            X = np.asarray(self.src.rows(new), np.float64)
            ids = np.concatenate([self.ids, new])
            Ht = np.concatenate([self.Ht, X @ self.W])
            order = np.argsort(ids, kind="stable")
            self.ids, self.Ht = ids[order], Ht[order]
        self.Al = (self.Ht.reshape(-1, self.h, self.f) * self.a_l).sum(-1)
        self.Ar = (self.Ht.reshape(-1, self.h, self.f) * self.a_r).sum(-1)

    def idx(self, ids):
        return np.searchsorted(self.ids, np.asarray(ids, np.int64))


def _row_softmax(T: _Tables, v: int, U: np.ndarray, slope):
    """alpha [len(U), h] and z of destination v's in-edges (rows of Ht indexed by U)."""
    if U.size == 0:
        return np.zeros((0, T.h)), np.zeros((0, T.h))
    z = T.Al[T.idx(U)] + T.Ar[T.idx([v])[0]]
    s = _lrelu(z, slope)
    p = np.exp(s - s.max(0))
    return p / p.sum(0), z


def gat_fwd_rows(src, W, a_l, a_r, h: int, f: int, rows, slope: float = 0.2) -> np.ndarray:
    """out[rows] in f64 ([len(rows), h*f])."""
    T = _Tables(src, W, a_l, a_r, h, f)
    nb = {int(v): np.asarray(src.in_nbrs(int(v)), np.int64) for v in rows}
    T.need(np.concatenate([np.asarray(rows, np.int64)] + list(nb.values())))
    out = np.zeros((len(rows), h * f))
    for i, v in enumerate(rows):
        U = nb[int(v)]
        if U.size == 0:
            continue
        a, _ = _row_softmax(T, v, U, slope)
        X = T.Ht[T.idx(U)].reshape(-1, h, f)
        out[i] = (a[:, :, None] * X).sum(0).reshape(-1)
    return out


def gat_bwd_rows(src, W, a_l, a_r, h: int, f: int, rows, slope: float = 0.2):
    """(dHt[rows], dH[rows]) in f64 for the sampled source rows."""
    T = _Tables(src, W, a_l, a_r, h, f)
    rows = [int(u) for u in rows]
    outs = {u: np.asarray(src.out_nbrs(u), np.int64) for u in rows}
    dsts = sorted(set(rows).union(*[set(o.tolist()) for o in outs.values()]))  # every v whose c[v] is needed
    ins = {v: np.asarray(src.in_nbrs(v), np.int64) for v in dsts}
    T.need(np.concatenate([np.asarray(dsts, np.int64)] + list(ins.values())))
    G = {v: np.asarray(g, np.float64).reshape(h, f) for v, g in zip(dsts, src.dout(np.asarray(dsts, np.int64)))}
    stats = {}  # v -> (alpha over in(v), z, dalpha, c)
    for v in dsts:
        U = ins[v]
        a, z = _row_softmax(T, v, U, slope)
        X = T.Ht[T.idx(U)].reshape(-1, h, f)
        da = (X * G[v]).sum(-1)
        stats[v] = (a, z, da, (a * da).sum(0))
    grad = lambda z: np.where(z > 0, 1.0, slope)  # noqa: E731
    dHt = np.zeros((len(rows), h * f))
    for i, u in enumerate(rows):
        acc = np.zeros((h, f))
        dAl = np.zeros(h)
        for v in np.unique(outs[u]):
            a, z, da, c = stats[int(v)]
            U = ins[int(v)]
            for j in np.nonzero(U == u)[0]:  # every parallel edge u -> v (multigraph)
                acc += a[j][:, None] * G[int(v)]
                dAl += grad(z[j]) * a[j] * (da[j] - c)
        a, z, da, c = stats[u]
        dAr = (grad(z) * a * (da - c)).sum(0) if a.size else np.zeros(h)
        dHt[i] = (acc + dAl[:, None] * T.a_l + dAr[:, None] * T.a_r).reshape(-1)
    return dHt, dHt @ T.W.T


def max_rel_err(a, b) -> float:
    """max |a-b| / max(1,|a|,|b|) (tensor.hpp:153-156)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if a.size == 0:
        return 0.0
    return float((np.abs(a - b) / np.maximum(1.0, np.maximum(np.abs(a), np.abs(b)))).max())


def max_norm_err(a, ref) -> float:
    """max |a-ref| / max(1, max|ref|): the gradient comparator at benchmark scale (DESIGN.md §2:
    sums over 10^5..10^9 terms in fp32 cannot meet the elementwise bound where entries cancel
    to near zero -- the reference's own f32 CPU port cannot either)."""
    a = np.asarray(a, np.float64)
    ref = np.asarray(ref, np.float64)
    if a.size == 0:
        return 0.0
    return float(np.abs(a - ref).max() / max(1.0, float(np.abs(ref).max())))


# ---------------------------------------------------------------------------
# Device-backed row sources and the model-level sampled check (tests/ and bench.py's
# checker leg): the GPU model's own layer inputs and outputs, fetched row by row.
# ---------------------------------------------------------------------------
class DeviceRows:
    """`src` for gat_fwd_rows / gat_bwd_rows over a DeviceGraph-like pair of indexes
    (csr_dst, csc_src with .off / .nbr device tensors) and device tensors H (layer input)
    and dOut (layer output gradient; None = all ones, the loss seed of SPEC.md:217)."""

    def __init__(self, csr, csc, H, dOut=None, hf=None):
        import torch

        self.torch = torch
        self.csr, self.csc, self.H, self.dOut, self.hf = csr, csc, H, dOut, hf
        self.doff = csr.off.cpu().numpy().view(np.uint64)
        self.soff = csc.off.cpu().numpy().view(np.uint64)

    def _slice(self, idx, off, i):
        a, b = int(off[i]), int(off[i + 1])
        return idx.nbr[a:b].cpu().numpy().view(np.uint32).astype(np.int64)

    def in_nbrs(self, v):
        return self._slice(self.csr, self.doff, int(v))

    def out_nbrs(self, u):
        return self._slice(self.csc, self.soff, int(u))

    def _rows(self, T, ids):
        t = self.torch
        ids = t.as_tensor(np.asarray(ids, np.int64), device=T.device)
        return T.index_select(0, ids).double().cpu().numpy()

    def rows(self, ids):
        return self._rows(self.H, ids)

    def dout(self, ids):
        if self.dOut is None:
            return np.ones((len(ids), self.hf))
        return self._rows(self.dOut, ids)


def gat_model_sampled_check(model, H, n_rows: int = 16, n_src: int = 4, seed: int = 0, dOut=None,
                            hub_src: bool = True) -> dict:
    """Sampled-row f64 parity of a models.GAT-like stack (layers with W, a_l, a_r, p.heads, p.f,
    p.slope; graph model.g with csr_dst / csc_src): one forward + backward on the device through
    the model's own path, then
      * out rows of the first and the last layer (destinations: the two largest in-degree
        rows -- split into edge-balance chunks -- the smallest, and random rows),
      * dH rows of the last layer's backward (its input gradient; sources: the largest
        out-degree row and random rows),
    each against the f64 local-neighbourhood restatement above, with the GPU's own layer
    input as the input.  Comparator: rel_err (tensor.hpp:153-156)."""
    import torch

    g = model.g
    V = g.num_vertices
    xs, stashes = model.forward(H)
    seed_grad = model.seed_grad(xs[-1]) if dOut is None else dOut
    grads = model.backward(xs, stashes, seed_grad)
    torch.cuda.synchronize()
    rng = np.random.default_rng(seed)
    din = np.diff(g.csr_dst.off.cpu().numpy().view(np.uint64).astype(np.int64))
    dout_deg = np.diff(g.csc_src.off.cpu().numpy().view(np.uint64).astype(np.int64))
    top = np.argsort(-din, kind="stable")[:2]
    rows = np.unique(np.concatenate([top, [int(np.argmin(din))], rng.integers(0, V, max(0, n_rows - 3))]))
    hub = [int(np.argmax(dout_deg))] if hub_src else []
    srcs = np.unique(np.concatenate([hub, rng.integers(0, V, max(0, n_src - len(hub)))]).astype(np.int64))
    res = {"rows_checked": {}, "max_rel_err": {}}
    for name, li in (("out_layer1", 0), ("out_last", len(model.layers) - 1)):
        L = model.layers[li]
        src = DeviceRows(g.csr_dst, g.csc_src, xs[li])
        ref = gat_fwd_rows(src, L.W.double().cpu().numpy(), L.a_l.double().cpu().numpy(),
                           L.a_r.double().cpu().numpy(), L.p.heads, L.p.f, rows, L.p.slope)
        got = xs[li + 1].index_select(0, torch.as_tensor(rows, device=H.device)).double().cpu().numpy()
        res["max_rel_err"][name] = max_rel_err(got, ref)
        res["rows_checked"][name] = int(rows.size)
    L = model.layers[-1]
    dO = None if dOut is None else dOut
    src = DeviceRows(g.csr_dst, g.csc_src, xs[-2], dO, hf=L.p.heads * L.p.f)
    _, dH = gat_bwd_rows(src, L.W.double().cpu().numpy(), L.a_l.double().cpu().numpy(), L.a_r.double().cpu().numpy(),
                         L.p.heads, L.p.f, srcs, L.p.slope)
    gdH = grads[-1].dH
    if gdH is not None:
        got = gdH.index_select(0, torch.as_tensor(srcs, device=H.device)).double().cpu().numpy()
        res["max_rel_err"]["dH_last"] = max_rel_err(got, dH)
        res["max_norm_err"] = {"dH_last": max_norm_err(got, dH)}
        res["rows_checked"]["dH_last"] = int(srcs.size)
    res["max_in_degree_checked"] = int(din[top[0]])
    res["max_out_degree_checked"] = int(dout_deg[srcs].max())
    return res
