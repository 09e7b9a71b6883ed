"""GPU parity of EdgeConv (bit-exact argmax) and GMMConv against the oracle."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2110_09524_b200 import DeviceGraph, edgeconv_backward, edgeconv_forward, gmm_backward, gmm_forward
from paper_2110_09524_b200.graph import knn_edges
from paper_2110_09524_b200.ops import edgeconv_region_forward

pytestmark = pytest.mark.gpu
TOL = 1e-4


def t32(x, dev):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(dev)


def np64(t):
    return t.detach().cpu().double().numpy()


# C picks K6/K7's column width per lane (VW) and lanes per row (L): 64 -> VW 8 / L 8 (4 rows per
# warp), 96 -> 8 / 16 with 4 idle lanes, 128 -> 8 / 16, 256 -> 8 / 32, 33 -> 1 / 32 with a partial
# second pass
@pytest.mark.parametrize("clouds,points,k,C", [(2, 256, 20, 64), (4, 1024, 40, 64), (1, 64, 8, 33),
                                               (2, 256, 20, 128), (1, 512, 16, 256), (2, 128, 10, 96)])
def test_edgeconv_region_argmax_bit_exact(cuda, clouds, points, k, C):
    src, dst = knn_edges(clouds, points, k, seed=0)
    V = clouds * points
    hg = O.host_graph(V, src, dst)
    g = DeviceGraph.from_edges(V, src, dst, device=cuda)
    rng = np.random.default_rng(C)
    # quantized values create exact ties, exercising the lowest-edge-id rule
    Th = (rng.integers(-8, 8, (V, C)) / 4.0).astype(np.float32)
    Ph = rng.uniform(-1, 1, (V, C)).astype(np.float32)
    ref_out, ref_amax = O.edgeconv_fwd(hg, Th, Ph, np.float32)
    out, amax = edgeconv_region_forward(g, t32(Th, cuda), t32(Ph, cuda))
    torch.cuda.synchronize()
    np.testing.assert_array_equal(amax.cpu().numpy().view(np.uint32), ref_amax)
    np.testing.assert_array_equal(out.cpu().numpy(), ref_out)  # same fp32 RN expression -> bitwise


@pytest.mark.parametrize("C", [8, 36, 64, 128, 200])
def test_edgeconv_ragged_rows(cuda, C):
    """Rows of different lengths (0 .. ~60 edges, some empty) side by side in one warp's lane groups:
    each group runs its own trip count.  Forward bitwise; backward against the f64 oracle routed by
    the shared argmax."""
    rng = np.random.default_rng(C + 7)
    V = 700
    deg = rng.integers(0, 60, V)
    deg[rng.random(V) < 0.1] = 0
    dst = np.repeat(np.arange(V), deg)
    src = rng.integers(0, V, dst.size)
    perm = rng.permutation(dst.size)  # edge ids not in row order
    src, dst = src[perm], dst[perm]
    hg = O.host_graph(V, src, dst)
    g = DeviceGraph.from_edges(V, src, dst, device=cuda)
    Th = (rng.integers(-8, 8, (V, C)) / 4.0).astype(np.float32)
    Ph = rng.uniform(-1, 1, (V, C)).astype(np.float32)
    ref_out, ref_amax = O.edgeconv_fwd(hg, Th, Ph, np.float32)
    out, amax = edgeconv_region_forward(g, t32(Th, cuda), t32(Ph, cuda))
    torch.cuda.synchronize()
    np.testing.assert_array_equal(amax.cpu().numpy().view(np.uint32), ref_amax)
    np.testing.assert_array_equal(out.cpu().numpy(), ref_out)
    Fin = 16
    H = rng.uniform(-1, 1, (V, Fin))
    Theta, Phi = rng.uniform(-0.25, 0.25, (Fin, C)), rng.uniform(-0.25, 0.25, (Fin, C))
    dOut = rng.uniform(-1, 1, (V, C))
    tH, tT, tP = t32(H, cuda), t32(Theta, cuda), t32(Phi, cuda)
    _, st = edgeconv_forward(g, tH, tT, tP)
    Y = st.Y.cpu().numpy()
    _, ref_amax2 = O.edgeconv_fwd(hg, Y[:, :C], Y[:, C:], np.float32)
    np.testing.assert_array_equal(st.argmax.cpu().numpy().view(np.uint32), ref_amax2)
    dH, dTheta, dPhi = edgeconv_backward(g, tH, tT, tP, st, t32(dOut, cuda))
    torch.cuda.synchronize()
    bw = O.edgeconv_layer_bwd_f64(hg, H, Theta, Phi, ref_amax2, dOut)
    for name, got in (("dH", dH), ("dTheta", dTheta), ("dPhi", dPhi)):
        scale = max(1.0, np.abs(bw[name]).max())
        assert O.max_rel_err(np64(got) / scale, bw[name] / scale) < TOL, name


def test_edgeconv_empty_rows_and_ties(cuda):
    src, dst = [1, 2, 3, 1, 2, 3], [0, 0, 0, 0, 0, 0]
    g = DeviceGraph.from_edges(4, src, dst, device=cuda)
    Th = t32([[0.0], [5.0], [5.0], [1.0]], cuda)
    out, amax = edgeconv_region_forward(g, Th, t32(np.zeros((4, 1)), cuda))
    a = amax.cpu().numpy().view(np.uint32)
    assert a[0, 0] == 0 and out[0, 0].item() == 5.0
    assert all(a[v, 0] == 0xFFFFFFFF and out[v, 0].item() == 0.0 for v in (1, 2, 3))


@pytest.mark.parametrize("k,C", [(20, 64), (40, 64), (20, 256), (12, 36)])
def test_edgeconv_layer_vs_oracle(cuda, k, C):
    src, dst = knn_edges(2, 512, k, seed=1)
    V = 1024
    hg = O.host_graph(V, src, dst)
    g = DeviceGraph.from_edges(V, src, dst, device=cuda)
    rng = np.random.default_rng(k)
    Fin = 64
    H = rng.uniform(-1, 1, (V, Fin))
    Theta, Phi = rng.uniform(-0.125, 0.125, (Fin, C)), rng.uniform(-0.125, 0.125, (Fin, C))
    dOut = rng.uniform(-1, 1, (V, C))
    tH, tT, tP = t32(H, cuda), t32(Theta, cuda), t32(Phi, cuda)
    out, st = edgeconv_forward(g, tH, tT, tP)
    # argmax parity is defined on identical Th/Ph: feed the device GEMM output to the f32 oracle
    Y = st.Y.cpu().numpy()
    ref_out, ref_amax = O.edgeconv_fwd(hg, Y[:, :C], Y[:, C:], np.float32)
    np.testing.assert_array_equal(st.argmax.cpu().numpy().view(np.uint32), ref_amax)
    np.testing.assert_array_equal(out.cpu().numpy(), ref_out)
    fw = O.edgeconv_layer_fwd_f64(hg, H, Theta, Phi)
    assert O.max_rel_err(np64(out), fw["out"]) < TOL
    dH, dTheta, dPhi = edgeconv_backward(g, tH, tT, tP, st, t32(dOut, cuda))
    torch.cuda.synchronize()
    bw = O.edgeconv_layer_bwd_f64(hg, H, Theta, Phi, ref_amax, dOut)  # route with the shared argmax
    for name, got in (("dH", dH), ("dTheta", dTheta), ("dPhi", dPhi)):
        scale = max(1.0, np.abs(bw[name]).max())
        assert O.max_rel_err(np64(got) / scale, bw[name] / scale) < TOL, name


# K f picks K8's lanes per row: <= 64 -> 8 (4 rows per warp), <= 128 -> 16, else 32
@pytest.mark.parametrize("V,E,Fin,K,r,f", [(200, 1500, 20, 3, 2, 16), (19717, 88648, 500, 3, 3, 16),
                                           (500, 4000, 8, 2, 1, 16), (300, 2000, 10, 8, 4, 32),
                                           (400, 6000, 12, 4, 3, 24), (350, 9000, 6, 1, 2, 5)])
def test_gmm_layer_vs_oracle(cuda, V, E, Fin, K, r, f):
    rng = np.random.default_rng(V)
    src, dst = rng.integers(0, V, E), rng.integers(0, V, E)
    hg = O.host_graph(V, src, dst)
    g = DeviceGraph.from_edges(V, src, dst, device=cuda)
    s = 1 / np.sqrt(Fin)
    H = rng.uniform(-1, 1, (V, Fin))
    W = rng.uniform(-s, s, (Fin, K * f))
    Pl, Pr = rng.uniform(-s, s, (Fin, r)), rng.uniform(-s, s, (Fin, r))
    mu, sinv = rng.uniform(-0.5, 0.5, (K, r)), rng.uniform(0.5, 1.5, (K, r))
    dOut = rng.uniform(-1, 1, (V, f))
    fw = O.gmm_layer_fwd_f64(hg, H, W, Pl, Pr, mu, sinv, K, r, f)
    bw = O.gmm_layer_bwd_f64(hg, H, W, Pl, Pr, mu, sinv, K, r, f, fw, dOut)
    args = [t32(x, cuda) for x in (H, W, Pl, Pr, mu, sinv)]
    out, st = gmm_forward(g, *args, K, r, f)
    grads = gmm_backward(g, *args, K, r, f, st, t32(dOut, cuda))
    torch.cuda.synchronize()
    assert O.max_rel_err(np64(out), fw["out"]) < TOL
    for name, got in zip(("dH", "dW", "dPl", "dPr", "dmu", "dsinv"), grads):
        scale = max(1.0, np.abs(bw[name]).max())
        assert O.max_rel_err(np64(got) / scale, bw[name] / scale) < TOL, name


def test_edgeless_graph_edgeconv_and_gmm(cuda):
    """E = 0 through EdgeConv (out 0, argmax = no edge) and GMMConv (out 0), forward and backward."""
    V, Fin, C, K, r, f = 29, 12, 16, 3, 2, 16
    g = DeviceGraph.from_edges(V, [], [], device=cuda)
    rng = np.random.default_rng(4)
    H = t32(rng.uniform(-1, 1, (V, Fin)), cuda)
    Th, Ph = t32(rng.uniform(-1, 1, (Fin, C)), cuda), t32(rng.uniform(-1, 1, (Fin, C)), cuda)
    out, st = edgeconv_forward(g, H, Th, Ph)
    grads = edgeconv_backward(g, H, Th, Ph, st, t32(rng.uniform(-1, 1, (V, C)), cuda))
    torch.cuda.synchronize()
    assert torch.count_nonzero(out) == 0
    assert bool((st.argmax == -1).all())  # 0xFFFFFFFF: empty row
    for t in grads:
        if t is not None:
            assert torch.count_nonzero(t) == 0
    args = [t32(x, cuda) for x in (rng.uniform(-1, 1, (V, Fin)), rng.uniform(-1, 1, (Fin, K * f)),
                                   rng.uniform(-1, 1, (Fin, r)), rng.uniform(-1, 1, (Fin, r)),
                                   rng.uniform(-0.5, 0.5, (K, r)), rng.uniform(0.5, 1.5, (K, r)))]
    o2, st2 = gmm_forward(g, *args, K, r, f)
    g2 = gmm_backward(g, *args, K, r, f, st2, t32(rng.uniform(-1, 1, (V, f)), cuda))
    torch.cuda.synchronize()
    assert torch.count_nonzero(o2) == 0
    for t in g2:
        if t is not None:
            assert torch.count_nonzero(t) == 0


@pytest.mark.parametrize("C", [64, 128, 256])
def test_edgeconv_column_alignment_paths_agree(cuda, C):
    """K6 / K7 pick 32-byte columns for aligned tables and 16 / 8 / 4-byte ones for shifted views
    (and with them the lanes per row); every column still walks its edges in the same order, so the
    outputs are bitwise equal across the paths."""
    from paper_2110_09524_b200._lib import call
    from paper_2110_09524_b200.graph import _ptr, _stream

    src, dst = knn_edges(2, 256, 20, seed=3)
    V = 512
    g = DeviceGraph.from_edges(V, src, dst, device=cuda)
    rng = np.random.default_rng(C)
    Th = t32((rng.integers(-8, 8, (V, C)) / 4.0).astype(np.float32), cuda)
    Ph = t32(rng.uniform(-1, 1, (V, C)), cuda)
    dOut = t32(rng.uniform(-1, 1, (V, C)), cuda)
    ref_out, ref_amax = edgeconv_region_forward(g, Th, Ph)

    def view(shift):
        return torch.zeros(V, C + 8, device=cuda)[:, shift:shift + C]

    def bwd(dTh, dPh):
        call("gnncg_edgeconv_bwd", g.csc_src.struct(), g.csr_dst.struct(), C, _ptr(ref_amax), _ptr(dOut), _ptr(dTh),
             dTh.stride(0), _ptr(dPh), dPh.stride(0), _stream())
        torch.cuda.synchronize()
        return dTh.clone(), dPh.clone()

    base = bwd(torch.empty(V, C, device=cuda), torch.empty(V, C, device=cuda))
    for shift in (1, 2, 4):  # 4 / 8 / 16-byte aligned rows
        bt, bp = view(shift), view(shift)
        bt.copy_(Th)
        bp.copy_(Ph)
        out, amax = edgeconv_region_forward(g, bt, bp)
        torch.cuda.synchronize()
        assert torch.equal(out, ref_out) and torch.equal(amax, ref_amax), shift
        d = bwd(view(shift), view(shift))
        assert torch.equal(d[0], base[0]) and torch.equal(d[1], base[1]), shift
