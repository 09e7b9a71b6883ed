"""CPU, world_size 2 and 3 over gloo: the multi-GPU orchestration of dist.py (row
partition, edges split by source owner, padded all-gather of Ht || A_l, the two-part forward
with its online-softmax merge, the two-pass backward whose remote partials are
reduce-scattered, dW / da all-reduced, SGD in lock-step) reproduces the single-process f64
oracle.

The product engine (CudaEngine + gnncg_gat_*_dist) cannot run here; the same PartitionedGAT
schedule is driven by an oracle-backed engine (test infrastructure) that restates
gnncg_gat_fwd_dist / gnncg_gat_bwd_dist per edge in numpy on the rank-local indexes.  The
GPU side of the same entry points is tested by tests/test_gpu_dist.py (world 1 over NCCL and
P ranks emulated on one GPU)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O


def merge2(A, B):
    """Online-softmax merge of two partials (out, m, d) of the same rows (gnncg_gat_fwd_dist)."""
    (oa, ma, da), (ob, mb, db) = A, B
    M = np.where(da == 0, mb, np.where(db == 0, ma, np.maximum(ma, mb)))
    ea = np.where(da == 0, 0.0, da * np.exp(ma - M))
    eb = np.where(db == 0, 0.0, db * np.exp(mb - M))
    D = ea + eb
    wa = np.divide(ea, D, out=np.zeros_like(D), where=D > 0)
    wb = np.divide(eb, D, out=np.zeros_like(D), where=D > 0)
    h = M.shape[1]
    f = oa.shape[1] // h
    out = (np.repeat(wa, f, 1) * oa + np.repeat(wb, f, 1) * ob)
    return out, M, D


class _Idx(dict):
    """An oracle-side index: the dict of O.build_index outputs, with num_edges as an attribute."""

    @property
    def num_edges(self):
        return self["num_edges"]


class OracleEngine:
    device = torch.device("cpu")

    def build_index(self, rows, key, other, n_other):
        key, other = key.numpy().astype(np.int64), other.numpy().astype(np.int64)
        assert key.size == 0 or (key.max() < rows and other.max() < n_other)
        off, nbr, eid = O.build_index(rows, key.astype(np.uint32), other.astype(np.uint32))
        return _Idx(off=off, nbr=nbr, eid=eid, rows=rows, num_edges=key.size)

    def zeros(self, *s):
        return torch.zeros(*s, dtype=torch.float64)

    empty = zeros

    def gemm(self, A, B, ta=False, tb=False, out=None):
        r = (A.T if ta else A) @ (B.T if tb else B)
        if out is None:
            return r
        out.copy_(r)
        return out

    def transform(self, H, W, a_l, a_r, p, Ht_out, Al_out):
        Ht = H @ W
        H3 = Ht.view(Ht.shape[0], p.heads, p.f)
        Ht_out.copy_(Ht)
        Al_out.copy_((H3 * a_l).sum(-1))
        return (H3 * a_r).sum(-1)

    @staticmethod
    def _edges(idx):
        """(v = local destination row, u = neighbour) of a csr index, in index order."""
        v = np.repeat(np.arange(idx["rows"]), np.diff(idx["off"].astype(np.int64)))
        return v, idx["nbr"].astype(np.int64)

    def _region(self, idx, Ht, Al, Ar, p):
        g = O.HostGraph(idx["rows"], None, None, idx["off"], idx["nbr"], idx["eid"], None, None, None)
        r = O.gat_region_fwd_f64(g, Ht, Al, Ar, p.heads, p.f, p.slope)
        return r["out"], r["m"], r["d"]

    def region_fwd(self, lg, Ht_all, Al_all, Ar, p):
        mr, b = lg.plan.maxrows, lg.row_base
        for t in (Ht_all, Al_all):  # the all-gather of the rank's block
            dist.all_gather_into_tensor(t, t[b:b + mr].clone())
        Ht, Al, Arn = Ht_all.numpy(), Al_all.numpy(), Ar.numpy()
        A = self._region(lg.csr_local, Ht, Al, Arn, p)
        B = self._region(lg.csr_remote, Ht, Al, Arn, p)
        return tuple(torch.from_numpy(x) for x in merge2(A, B))

    def region_bwd(self, lg, Ht_all, Al_all, Ar, m, d, out, dOut, a_l, a_r, p):
        h, f, n, b, mr, Vp = p.heads, p.f, lg.num_local, lg.row_base, lg.plan.maxrows, lg.plan.padded_V
        Ht3, Al, Arn = Ht_all.numpy().reshape(-1, h, f), Al_all.numpy(), Ar.numpy()
        dO3, mn, dn = dOut.numpy().reshape(n, h, f), m.numpy(), d.numpy()
        al, ar = a_l.numpy(), a_r.numpy()

        def edge_terms(idx):
            v, u = self._edges(idx)
            z = Al[u] + Arn[v]
            a = np.exp(np.where(z > 0, z, p.slope * z) - mn[v]) / dn[v]
            da = (dO3[v] * Ht3[u]).sum(-1)
            return v, u, z, a, da

        parts = [edge_terms(lg.csr_remote), edge_terms(lg.csr_local)]
        c = np.zeros((n, h))
        for v, u, z, a, da in parts:  # c[v] over ALL in-edges of v (both parts)
            np.add.at(c, v, a * da)
        dAr = np.zeros((n, h))
        outs = []
        for (v, u, z, a, da), rows, shift in zip(parts, (Vp, n), (0, b)):
            dz = np.where(z > 0, 1.0, p.slope) * a * (da - c[v])
            dHt, dAl = np.zeros((rows, h, f)), np.zeros((rows, h))
            np.add.at(dAl, u - shift, dz)
            np.add.at(dAr, v, dz)
            np.add.at(dHt, u - shift, a[:, :, None] * dO3[v])
            dHt += dAl[:, :, None] * al[None]
            outs.append((dHt.reshape(rows, h * f), dAl))
        (sendH, sendAl), (ownH, ownAl) = outs
        recvH, recvAl = torch.zeros(mr, h * f, dtype=torch.float64), torch.zeros(mr, h, dtype=torch.float64)
        dist.reduce_scatter_tensor(recvH, torch.from_numpy(sendH))
        dist.reduce_scatter_tensor(recvAl, torch.from_numpy(sendAl))
        dHt = ownH + recvH.numpy()[:n] + np.repeat(dAr, f, 1) * ar.reshape(1, h * f)
        dAl = ownAl + recvAl.numpy()[:n]
        return torch.from_numpy(dHt), torch.from_numpy(dAl), torch.from_numpy(dAr)

    def attn_grad(self, Ht, dAl, dAr, p, out=None):
        H3 = Ht.reshape(-1, p.heads, p.f)
        r = ((dAl[:, :, None] * H3).sum(0), (dAr[:, :, None] * H3).sum(0))
        if out is None:
            return r
        for o, x in zip(out, r):
            o.copy_(x)
        return out

    def all_reduce(self, t):
        dist.all_reduce(t)
        return t

    def sgd(self, param, grad, lr):
        param -= lr * grad

    def fill_ones(self, like):
        return torch.ones_like(like)

    def total(self, x, out):
        out[0] = x.sum()


def _pairs(idx, transpose=False):
    v, u = OracleEngine._edges(idx)
    return sorted(zip(u.tolist(), v.tolist())) if transpose else sorted(zip(v.tolist(), u.tolist()))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2110_09524_b200.dist import PartitionedGAT, PartitionPlan, build_local

        V, src, dst, H, params, dims = case
        eng = OracleEngine()
        plan = PartitionPlan.from_dst(V, torch.from_numpy(dst.astype(np.int64)), world)
        lg = build_local(plan, rank, torch.from_numpy(src.astype(np.int64)), torch.from_numpy(dst.astype(np.int64)),
                         eng)
        # the csc indexes are the transposes of the csr ones (csc_local rows rebased to the block)
        base = lg.row_base
        assert _pairs(lg.csr_remote) == sorted(_pairs(lg.csc_remote, transpose=True))
        assert _pairs(lg.csr_local) == sorted((v, u + base) for v, u in _pairs(lg.csc_local, transpose=True))
        assert all(base <= u < base + lg.num_local for _, u in _pairs(lg.csr_local))
        assert not any(base <= u < base + lg.num_local for _, u in _pairs(lg.csr_remote))
        assert lg.num_edges == int((dst >= plan.bounds[rank]).sum() - (dst >= plan.bounds[rank + 1]).sum())
        r0, r1 = int(plan.bounds[rank]), int(plan.bounds[rank + 1])
        tparams = [tuple(torch.from_numpy(x.copy()) for x in p) for p in params]
        model = PartitionedGAT(lg, dims, engine=eng, params=tparams)
        xs, stashes = model.forward(torch.from_numpy(H[r0:r1].copy()))
        loss = xs[-1].sum().clone()
        dist.all_reduce(loss)
        grads = model.backward(xs, stashes, torch.ones_like(xs[-1]))
        q.put((rank, r0, r1, xs[-1].numpy(), float(loss), [tuple(g[j].numpy() for j in range(3)) for g in grads]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_partitioned_gat_matches_single_process_oracle(world):
    rng = np.random.default_rng(world)
    V, E = 120, 1500
    w = 1.0 / (np.arange(V) + 5.0)
    w /= w.sum()
    src, dst = rng.choice(V, E, p=w), rng.choice(V, E, p=w)
    dims = [(12, 2, 4), (8, 2, 4)]
    H = rng.uniform(-1, 1, (V, 12))
    params = [(rng.uniform(-0.5, 0.5, (fin, h * f)), rng.uniform(-0.5, 0.5, (h, f)), rng.uniform(-0.5, 0.5, (h, f)))
              for fin, h, f in dims]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, (V, src, dst, H, params, dims), q)) for r in range(world)]
    for p in procs:
        p.start()
    import queue
    import time

    res, t0 = [], time.time()
    while len(res) < world:  # fail fast when a rank dies instead of waiting out the queue
        try:
            res.append(q.get(timeout=2))
        except queue.Empty:
            dead = [p.exitcode for p in procs if p.exitcode not in (None, 0)]
            assert not dead and time.time() - t0 < 300, f"rank exit codes {dead}"
    res.sort(key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    hg = O.host_graph(V, src, dst)
    f1 = O.gat_layer_fwd_f64(hg, H, *params[0], 2, 4)
    f2 = O.gat_layer_fwd_f64(hg, f1["out"], *params[1], 2, 4)
    b2 = O.gat_layer_bwd_f64(hg, f1["out"], *params[1], 2, 4, f2, np.ones((V, 8)))
    b1 = O.gat_layer_bwd_f64(hg, H, *params[0], 2, 4, f1, b2["dH"], need_dH=False)
    out = np.zeros((V, 8))
    for rank, r0, r1, o, loss, grads in res:
        out[r0:r1] = o
        assert abs(loss - f2["out"].sum()) < 1e-9
        for (dW, dal, dar), b in zip(grads, (b1, b2)):
            np.testing.assert_allclose(dW, b["dW"], atol=1e-10)
            np.testing.assert_allclose(dal, b["dal"], atol=1e-10)
            np.testing.assert_allclose(dar, b["dar"], atol=1e-10)
    np.testing.assert_allclose(out, f2["out"], atol=1e-12)
    assert sorted((r0, r1) for _, r0, r1, *_ in res)[-1][1] == V
