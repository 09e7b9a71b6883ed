"""GPU: the two lane layouts of the lean 8 x 32 kernels (gat_lean.cu) -- 256-bit lane rows for
32-byte aligned tables, the paired 2 x 128-bit layout for tables that are only 16-byte aligned
(a caller's column view or offset pointer) -- give the same results: K2 bitwise (same per-column
accumulation order), K4f up to the order of its head-dot reductions and dA_r sums."""
import numpy as np
import pytest
import torch

from paper_2110_09524_b200 import DeviceGraph, GatParams
from paper_2110_09524_b200.ops import GatStash, gat_region_backward, gat_region_forward

pytestmark = pytest.mark.gpu


def _offset_copy(t, floats):
    """The same values at a storage offset of `floats` floats (16-byte aligned for floats = 4)."""
    buf = torch.empty(t.numel() + floats, dtype=t.dtype, device=t.device)
    v = buf[floats:].view_as(t)
    v.copy_(t)
    return v


@pytest.mark.parametrize("kind", ["powerlaw", "hubs"])
def test_aligned_and_16b_tables_agree(cuda, kind):
    dev = torch.device("cuda:0")
    if kind == "powerlaw":
        g = DeviceGraph.chung_lu(6000, 400_000, offset=50, seed=5, device=dev)
    else:  # split rows (> 2048 edges) in both directions
        rng = np.random.default_rng(1)
        V = 5000
        src = np.concatenate([rng.integers(0, V, 6000), np.full(5000, 3)])
        dst = np.concatenate([np.zeros(6000, np.int64), rng.integers(0, V, 5000)])
        g = DeviceGraph.from_edges(V, src, dst, device=dev)
    V, h, f = g.num_vertices, 8, 32
    gen = torch.Generator(device=dev).manual_seed(0)
    u = lambda *s: torch.rand(*s, device=dev, generator=gen) * 2 - 1  # noqa: E731
    Ht, Al, Ar, al, ar, dOut = u(V, h * f), u(V, h), u(V, h), u(h, f), u(h, f), u(V, h * f)
    p = GatParams(h, f)
    res = []
    for off in (0, 4):
        tHt = Ht if off == 0 else _offset_copy(Ht, off)
        tdO = dOut if off == 0 else _offset_copy(dOut, off)
        assert (tHt.data_ptr() % 32 == 0) == (off == 0) and tdO.data_ptr() % 16 == 0
        out, m, d = gat_region_forward(g, tHt, Al, Ar, p)
        st = GatStash(tHt, Al, Ar, m, d, out)
        dHt, dAl, dAr, *_ = gat_region_backward(g, st, al, ar, tdO, p, mode="fast")
        torch.cuda.synchronize()
        res.append([x.cpu().numpy() for x in (out, m, d, dHt, dAl, dAr)])
    a, b = res
    for x, y in zip(a[:3], b[:3]):
        np.testing.assert_array_equal(x, y)
    for x, y in zip(a[3:], b[3:]):
        s = max(1.0, float(np.abs(x).max()))
        assert float(np.abs(x - y).max()) / s < 1e-5
