"""GPU: the L2-persisting window over the hottest gathered rows (gnncg_l2_persist +
gnncg_sched_t.gather_off) is a cache policy only -- K2's outputs are bitwise identical with it
on, K4f's gradients equal up to the order of its dA_r reductions -- and every entry point that
takes a schedule still works when the hint is absent (dist indexes, C++ callers)."""
import numpy as np
import pytest
import torch

from paper_2110_09524_b200 import DeviceGraph, GatParams, _lib
from paper_2110_09524_b200.ops import GatStash, gat_region_backward, gat_region_forward

pytestmark = pytest.mark.gpu


def _run(g, h, f, seed=0):
    dev = g.device
    gen = torch.Generator(device=dev).manual_seed(seed)
    V = g.num_vertices
    u = lambda *s: torch.rand(*s, device=dev, generator=gen) * 2 - 1  # noqa: E731
    Ht, Al, Ar, al, ar, dOut = u(V, h * f), u(V, h), u(V, h), u(h, f), u(h, f), u(V, h * f)
    p = GatParams(h, f)
    out, m, d = gat_region_forward(g, Ht, Al, Ar, p)
    st = GatStash(Ht, Al, Ar, m, d, out)
    dHt, dAl, dAr, *_ = gat_region_backward(g, st, al, ar, dOut, p, mode="fast")
    torch.cuda.synchronize()
    return [x.cpu().numpy() for x in (out, m, d, dHt, dAl, dAr)]


@pytest.mark.parametrize("h,f", [(8, 32), (8, 16)])
def test_l2_window_is_cache_policy_only(cuda, h, f):
    g = DeviceGraph.chung_lu(20_000, 1_500_000, offset=100, seed=3, device="cuda")
    assert g.csr_dst.sched().struct().gather_rows == 20_000
    try:
        _lib.l2_persist(0)
        a = _run(g, h, f)
        got = _lib.l2_persist(8 << 20)
        assert 0 < got <= 8 << 20
        b = _run(g, h, f)
    finally:
        _lib.l2_persist(0)
    for x, y in zip(a[:3], b[:3]):  # forward: same items, same order per item
        np.testing.assert_array_equal(x, y)
    for x, y in zip(a[3:], b[3:]):  # K4f: dA_r sums arrive in any order
        s = max(1.0, float(np.abs(x).max()))
        assert float(np.abs(x - y).max()) / s < 1e-6


def test_degree_relabel_is_a_renaming(cuda):
    """DeviceGraph.relabel(degree_order()) renames vertices only: the GAT region on the relabeled
    graph with permuted inputs gives the permuted outputs (bitwise forward: edge ids and per-row
    edge order are unchanged), and the hottest rows land at the low ids."""
    from paper_2110_09524_b200 import permute_rows, unpermute_rows

    g0 = DeviceGraph.chung_lu(20_000, 1_000_000, offset=100, seed=4, device="cuda")
    shuffle = torch.randperm(20_000, generator=torch.Generator().manual_seed(1)).to("cuda")
    g = g0.relabel(shuffle)  # an arbitrary labelling
    perm = g.degree_order()
    gr = g.relabel(perm)
    deg = lambda x: (x.csr_dst.off[1:] - x.csr_dst.off[:-1]) + (x.csc_src.off[1:] - x.csc_src.off[:-1])  # noqa: E731
    d = deg(gr)
    assert bool((d[:-1] >= d[1:]).all())  # descending
    assert torch.equal(torch.sort(deg(g)).values, torch.sort(d).values)
    h, f = 8, 32
    gen = torch.Generator(device="cuda").manual_seed(3)
    u = lambda *s: torch.rand(*s, device="cuda", generator=gen) * 2 - 1  # noqa: E731
    Ht, Al, Ar, dOut = u(20_000, h * f), u(20_000, h), u(20_000, h), u(20_000, h * f)
    al, ar = u(h, f), u(h, f)
    p = GatParams(h, f)
    out, m, dd = gat_region_forward(g, Ht, Al, Ar, p)
    P = lambda x: permute_rows(x, perm)  # noqa: E731
    out2, m2, d2 = gat_region_forward(gr, P(Ht), P(Al), P(Ar), p)
    for x, y in ((out, out2), (m, m2), (dd, d2)):
        assert torch.equal(x, unpermute_rows(y, perm))
    st = GatStash(Ht, Al, Ar, m, dd, out)
    st2 = GatStash(P(Ht), P(Al), P(Ar), m2, d2, out2)
    a = gat_region_backward(g, st, al, ar, dOut, p, mode="fast")
    b = gat_region_backward(gr, st2, al, ar, P(dOut), p, mode="fast")
    for x, y in zip(a[:3], b[:3]):  # dHt, dA_l, dA_r
        y = unpermute_rows(y, perm)
        s = max(1.0, float(x.abs().max()))
        assert float((x - y).abs().max()) / s < 1e-5
