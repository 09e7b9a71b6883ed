"""GPU parity of the GCN path (weighted Aggregate, csrc/spmm.cu) against the oracle:
the aggregate forward and transposed, the layer forward/backward in f64, the symmetric
normalisation (bit-exact), and the training smoke of SPEC.md:368."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2110_09524_b200 import DeviceGraph, gcn_backward, gcn_forward, gcn_norm, spmm
from paper_2110_09524_b200.models import GCN
from tests.test_gpu_gat import make_graph, np64, t32

pytestmark = pytest.mark.gpu
TOL = 1e-4


@pytest.mark.parametrize("kind", ["G3", "ER16", "cora", "star", "powerlaw"])
@pytest.mark.parametrize("cols", [1, 3, 6, 64, 256, 602, 1030])
@pytest.mark.parametrize("transpose", [False, True])
def test_spmm_vs_oracle(cuda, kind, cols, transpose):
    hg, g = make_graph(kind, cuda)
    rng = np.random.default_rng(cols)
    X = rng.uniform(-1, 1, (hg.V, cols)).astype(np.float32)
    w = rng.uniform(-1, 1, hg.E).astype(np.float32)
    b = rng.uniform(-1, 1, cols).astype(np.float32)
    for chunk in (None, 64):
        for weighted, bias, relu in ((False, False, False), (True, True, True)):
            ref = O.gcn_aggregate(hg, X, w if weighted else None, b if bias else None, relu, transpose)
            got = spmm(g, t32(X, cuda), t32(w, cuda) if weighted else None, t32(b, cuda) if bias else None, relu,
                       transpose=transpose, chunk=chunk)
            assert O.max_rel_err(np64(got), ref) < TOL, (chunk, weighted)


def test_spmm_empty_graph_and_limits(cuda):
    g = DeviceGraph.from_edges(5, [], [], device=cuda)
    X = torch.ones(5, 8, device=cuda)
    assert torch.count_nonzero(spmm(g, X)).item() == 0
    b = torch.arange(8, dtype=torch.float32, device=cuda)
    out = spmm(g, X, bias=b, relu=True)
    assert torch.equal(out, b.expand(5, 8))  # empty rows: act(bias)
    hg, g = make_graph("ER16", cuda)
    X = torch.rand(16, 2500, device=cuda)  # several column tiles
    ref = O.gcn_aggregate(hg, X.cpu().numpy())
    assert O.max_rel_err(np64(spmm(g, X)), ref) < TOL


@pytest.mark.parametrize("kind", ["G3", "ER16", "star", "powerlaw"])
def test_gcn_norm_bit_exact(cuda, kind):
    hg, g = make_graph(kind, cuda)
    np.testing.assert_array_equal(gcn_norm(g).cpu().numpy(), O.gcn_norm(hg))


@pytest.mark.parametrize("kind,Fin,C", [("G3", 3, 4), ("ER16", 5, 8), ("cora", 64, 32), ("star", 48, 64),
                                        ("powerlaw", 602, 256)])
def test_gcn_layer_vs_oracle(cuda, kind, Fin, C):
    hg, g = make_graph(kind, cuda)
    rng = np.random.default_rng(Fin)
    H = rng.uniform(-1, 1, (hg.V, Fin))
    W = rng.uniform(-1, 1, (Fin, C)) / np.sqrt(Fin)
    b = rng.uniform(-0.5, 0.5, C)
    dOut = rng.uniform(-1, 1, (hg.V, C))
    w = O.gcn_norm(hg)
    H32, W32, b32, dO32 = (t32(x, cuda) for x in (H, W, b, dOut))
    # the oracle runs on the fp32-rounded inputs so only arithmetic differs
    H, W, b, dOut = (x.astype(np.float32).astype(np.float64) for x in (H, W, b, dOut))
    fw = O.gcn_layer_fwd_f64(hg, H, W, b, w.astype(np.float64))
    out, st = gcn_forward(g, H32, W32, b32, gcn_norm(g))
    dH, dW, db = gcn_backward(g, H32, W32, st, dO32, gcn_norm(g))
    assert O.max_rel_err(np64(out), fw["out"]) < TOL
    # the backward is checked given the forward's stash: the ReLU mask is the device output's
    # (a z within fp32 rounding of 0 may legitimately fall either side)
    bw = O.gcn_layer_bwd_f64(hg, H, W, {"out": np64(out)}, dOut, w.astype(np.float64))
    for name, got in (("dH", dH), ("dW", dW), ("db", db)):
        scale = max(1.0, np.abs(bw[name]).max())  # reductions over V: compare relative to the magnitude
        assert O.max_rel_err(np64(got) / scale, bw[name] / scale) < TOL, name


def test_gcn_training_loss_decreases(cuda):
    # GCN on k_regular_in(V=32, k=4), lr = 1e-3, 10 steps -> loss decreases
    V, k = 32, 4
    dst = np.repeat(np.arange(V), k)
    src = (dst + np.tile(np.arange(1, k + 1), V)) % V
    g = DeviceGraph.from_edges(V, src, dst, device=cuda)
    model = GCN(g, [8, 8, 4], seed=42)
    H = torch.rand(V, 8, generator=torch.Generator(device=cuda).manual_seed(1), device=cuda)
    losses = [model.train_step(H, lr=1e-3)[0].item() for _ in range(10)]
    assert losses[-1] < losses[0]
    assert all(np.isfinite(losses))
