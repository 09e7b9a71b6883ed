"""GPU: the partitioned (multi-GPU) GAT path through the library's own entry points.

Only one GPU is available per box here, so two things are checked separately:
  * P ranks EMULATED on one GPU: gnncg_gat_fwd_dist / gnncg_gat_bwd_dist with comm = NULL
    for every rank of a P-way partition (P = 2, 3, 8), the all-gather done by the test
    (the padded tables filled from the single-GPU Ht / A_l) and the reduce-scatter done by
    the test (the ranks' remote partials summed).  The rows of every rank must equal the
    single-GPU region forward / fused backward on the whole graph -- this runs the
    local / remote split, the online-softmax merge, both K4f passes and the combine of
    the C code at P > 1;
  * world size 1 over NCCL: the library's communicator (gnncg_comm_*, NCCL resolved at run
    time) driving PartitionedGAT step for step against the single-GPU model.
The world-size 2/3 orchestration over real collectives is covered on CPU by
tests/test_dist_gloo.py."""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture(scope="module")
def nccl_world1(cuda):
    if not dist.is_initialized():
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_port()}", rank=0, world_size=1,
                                device_id=cuda)
    yield
    dist.destroy_process_group()


def _rel(a, b):
    a, b = a.double().cpu().numpy(), b.double().cpu().numpy()
    return O.max_rel_err(a, b)


def _norm(a, b):
    a, b = a.double().cpu().numpy(), b.double().cpu().numpy()
    s = max(1.0, float(np.abs(b).max()))
    return float(np.abs(a - b).max()) / s


@pytest.mark.parametrize("P", [2, 3, 8])
@pytest.mark.parametrize("hf", [(8, 16), (8, 32)])
def test_emulated_ranks_match_single_gpu_region(cuda, P, hf):
    from paper_2110_09524_b200.dist import CudaEngine, partitioned_chung_lu
    from paper_2110_09524_b200.graph import DeviceGraph
    from paper_2110_09524_b200.ops import GatParams, GatStash, gat_region_backward, gat_region_forward

    h, f = hf
    V, E = 6000, 400_000  # hub rows above the 2048-edge split on every rank
    g = DeviceGraph.chung_lu(V, E, offset=40, seed=3, device=cuda)
    gen = torch.Generator(device=cuda)
    gen.manual_seed(11)
    Ht = torch.rand(V, h * f, generator=gen, device=cuda) * 2 - 1
    Al = torch.rand(V, h, generator=gen, device=cuda) * 2 - 1
    Ar = torch.rand(V, h, generator=gen, device=cuda) * 2 - 1
    dOut = torch.rand(V, h * f, generator=gen, device=cuda) * 2 - 1
    a_l = torch.rand(h, f, generator=gen, device=cuda) - 0.5
    a_r = torch.rand(h, f, generator=gen, device=cuda) - 0.5
    p = GatParams(h, f)
    out, m, d = gat_region_forward(g, Ht, Al, Ar, p)
    dHt, dAl, dAr, *_ = gat_region_backward(g, GatStash(Ht, Al, Ar, m, d, out), a_l, a_r, dOut, p, mode="fast")

    ranks = [partitioned_chung_lu(V, E, offset=40, seed=3, rank=r, world=P, device=cuda) for r in range(P)]
    plan = ranks[0].plan
    mr = plan.maxrows
    # the all-gather, done here: rank q's rows at [q*mr, q*mr + n_q)
    Ht_all = torch.zeros(P * mr, h * f, device=cuda)
    Al_all = torch.zeros(P * mr, h, device=cuda)
    for q in range(P):
        r0, r1 = int(plan.bounds[q]), int(plan.bounds[q + 1])
        Ht_all[q * mr:q * mr + r1 - r0] = Ht[r0:r1]
        Al_all[q * mr:q * mr + r1 - r0] = Al[r0:r1]
    eng = CudaEngine(cuda)  # comm = None
    sends, owned = [], []
    for q, lg in enumerate(ranks):
        r0, r1 = int(plan.bounds[q]), int(plan.bounds[q + 1])
        assert lg.csr_remote.num_edges > 0 and lg.csr_local.num_edges > 0
        o, mq, dq = eng.region_fwd(lg, Ht_all, Al_all, Ar[r0:r1].contiguous(), p)
        assert _rel(o, out[r0:r1]) < 1e-5 and _rel(mq, m[r0:r1]) < 1e-6 and _rel(dq, d[r0:r1]) < 1e-5
        hs, als = torch.empty(P * mr, h * f, device=cuda), torch.empty(P * mr, h, device=cuda)
        got = eng.region_bwd(lg, Ht_all, Al_all, Ar[r0:r1].contiguous(), mq, dq, o, dOut[r0:r1].contiguous(), a_l,
                             a_r, p, send=(hs, als))
        sends.append((hs, als))
        owned.append(got)
    # the reduce-scatter, done here
    sumH = sum(s[0] for s in sends)
    sumAl = sum(s[1] for s in sends)
    for q in range(P):
        r0, r1 = int(plan.bounds[q]), int(plan.bounds[q + 1])
        gH, gAl, gAr = owned[q]
        assert float(sends[q][0][q * mr:(q + 1) * mr].abs().max()) == 0.0  # own block: no remote partial
        eH = _norm(gH + sumH[q * mr:q * mr + r1 - r0], dHt[r0:r1])
        eAl = _norm(gAl + sumAl[q * mr:q * mr + r1 - r0], dAl[r0:r1])
        eAr = _norm(gAr, dAr[r0:r1])
        assert max(eH, eAl, eAr) < 1e-5, (q, eH, eAl, eAr)
    torch.cuda.synchronize()


def test_comm_world1_collectives(cuda, nccl_world1):
    from paper_2110_09524_b200 import _lib
    from paper_2110_09524_b200.dist import NcclComm
    from paper_2110_09524_b200.graph import _ptr, _stream

    comm = NcclComm()
    L = _lib.lib()
    assert L.gnncg_comm_size(comm.handle) == 1 and L.gnncg_comm_rank(comm.handle) == 0
    x = torch.arange(1000, dtype=torch.float32, device=cuda)
    y = torch.empty_like(x)
    _lib.call("gnncg_comm_allgather", comm.handle, _ptr(x), _ptr(y), x.numel(), _stream())
    z = torch.empty_like(x)
    _lib.call("gnncg_comm_reduce_scatter", comm.handle, _ptr(y), _ptr(z), x.numel(), _stream())
    comm.all_reduce(z)
    torch.cuda.synchronize()
    assert torch.equal(y, x) and torch.equal(z, x)
    comm.close()


def test_comm_rejects_bad_arguments(cuda):
    from paper_2110_09524_b200 import _lib

    L = _lib.lib()
    h = C.c_void_p()
    assert L.gnncg_comm_init(C.byref(h), 2, 5, C.create_string_buffer(128)) == 7  # rank out of range
    assert L.gnncg_comm_allgather(None, None, None, 4, None) == 7


def test_partitioned_world1_matches_single_gpu(cuda, nccl_world1):
    from paper_2110_09524_b200.dist import PartitionedGAT, partitioned_chung_lu
    from paper_2110_09524_b200.graph import DeviceGraph
    from paper_2110_09524_b200.models import GAT

    V, E, dims = 3000, 120_000, [(64, 8, 16), (128, 8, 16)]
    lg = partitioned_chung_lu(V, E, offset=40, seed=5, rank=0, world=1, device=cuda)
    pm = PartitionedGAT(lg, dims, seed=7)  # engine over the library's NCCL communicator (world 1)
    assert pm.engine.comm is not None
    g = DeviceGraph.chung_lu(V, E, offset=40, seed=5, device=cuda)
    sm = GAT(g, dims, seed=7)
    gen = torch.Generator(device=cuda)
    gen.manual_seed(3)
    H = torch.rand(V, 64, generator=gen, device=cuda) * 2 - 1
    xs_p, _ = pm.forward(H)
    xs_s, _ = sm.forward(H)
    assert _rel(xs_p[-1], xs_s[-1]) < 1e-5
    lp, gp = pm.train_step(H, lr=0.0)
    ls, gs = sm.train_step(H, lr=0.0)
    torch.cuda.synchronize()
    assert abs(lp.item() - ls.item()) <= 1e-4 * max(1.0, abs(ls.item()))
    for (dW, da_l, da_r, _), gr in zip(gp, gs):
        for a, b in ((dW, gr.dW), (da_l, gr.da_l), (da_r, gr.da_r)):
            assert _norm(a, b) < 1e-4
    pm.engine.comm.close()


def test_part_bounds_are_validated(cuda):
    """gnncg_part_t.bounds (the owned-rows collectives) must agree with num_local and maxrows:
    a part whose bounds disagree is refused with GNNCG_ERR_ARG instead of moving wrong rows."""
    from paper_2110_09524_b200 import _lib
    from paper_2110_09524_b200.dist import CudaEngine, partitioned_chung_lu
    from paper_2110_09524_b200.graph import _ptr, _stream

    lg = partitioned_chung_lu(3000, 100_000, offset=40, seed=3, rank=1, world=2, device=cuda)
    eng = CudaEngine(cuda)
    pt = eng.part(lg)
    h, f = 8, 16
    n, mr = lg.num_local, lg.plan.maxrows
    Ht_all = torch.zeros(2 * mr, h * f, device=cuda)
    Al_all = torch.zeros(2 * mr, h, device=cuda)
    Ar = torch.zeros(n, h, device=cuda)
    out = torch.empty(n, h * f, device=cuda)
    m, d = torch.empty(n, h, device=cuda), torch.empty(n, h, device=cuda)
    ws = torch.empty(_lib.lib().gnncg_gat_dist_workspace(C.byref(pt), h, f), dtype=torch.uint8, device=cuda)
    args = lambda: (None, C.byref(pt), h, f, 0.2, _ptr(Ht_all), _ptr(Al_all), _ptr(Ar), _ptr(out), _ptr(m),  # noqa: E731
                    _ptr(d), _ptr(ws), ws.numel(), _stream())
    _lib.call("gnncg_gat_fwd_dist", *args())  # consistent bounds: accepted
    bad = np.ascontiguousarray(lg.plan.bounds, dtype=np.uint64).copy()
    bad[1] += 1  # rank 1's block no longer matches num_local
    pt.bounds = bad.ctypes.data
    with pytest.raises(_lib.ArgumentError):
        _lib.call("gnncg_gat_fwd_dist", *args())
