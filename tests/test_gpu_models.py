"""GPU: the model steps the bench runs for configs[0,2,3] and the GCN row (models.EdgeConvNet,
models.MoNet, models.GCN) -- parameter buffers with column views ([Theta | Phi],
[W | P_l | P_r | 0]), loss, backward and SGD -- against the f64 oracle layer by layer, eagerly
and replayed as a CUDA graph (models.GraphedStep), on graphs of the bench generators."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2110_09524_b200.graph import DeviceGraph, knn_edges, uniform_edges
from paper_2110_09524_b200.models import GCN, EdgeConvNet, GraphedStep, MoNet

pytestmark = pytest.mark.gpu


def np64(t):
    return t.detach().double().cpu().numpy()


def norm_err(a, b):
    s = max(1.0, float(np.abs(b).max()))
    return float(np.abs(a - b).max()) / s


def feats(V, F, dev, seed=5):
    gen = torch.Generator(device=dev)
    gen.manual_seed(seed)
    ld = (F + 3) // 4 * 4
    return (torch.rand(V, ld, generator=gen, device=dev) * 2 - 1)[:, :F]


def test_edgeconv_net_step_matches_oracle(cuda):
    src, dst = knn_edges(2, 256, 10, seed=1)
    V = 512
    g = DeviceGraph.from_edges(V, src, dst, device=cuda)
    dims = [16, 32, 32]
    model = EdgeConvNet(g, dims, seed=2)
    params0 = [np64(W) for W in model.layers]
    H = feats(V, 16, cuda)
    loss, grads = model.train_step(H, lr=0.0)
    torch.cuda.synchronize()
    hg = O.host_graph(V, src, dst)
    xs, fws = [np64(H)], []
    for Wc in params0:
        C = Wc.shape[1] // 2
        fw = O.edgeconv_layer_fwd_f64(hg, xs[-1], Wc[:, :C], Wc[:, C:])
        fws.append(fw)
        xs.append(fw["out"])
    assert abs(float(loss.item()) - xs[-1].sum()) <= 1e-4 * max(1.0, abs(xs[-1].sum()))
    gr = np.ones_like(xs[-1])
    for i in reversed(range(len(params0))):
        Wc = params0[i]
        C = Wc.shape[1] // 2
        bw = O.edgeconv_layer_bwd_f64(hg, xs[i], Wc[:, :C], Wc[:, C:], fws[i]["amax"], gr, need_dH=i > 0)
        dTh, dPh = grads[i]
        assert norm_err(np64(dTh), bw["dTheta"]) < 1e-4 and norm_err(np64(dPh), bw["dPhi"]) < 1e-4
        gr = bw["dH"]


def test_monet_step_matches_oracle(cuda):
    V, E, K, r = 3000, 20000, 3, 3
    src, dst = uniform_edges(V, E, seed=3)
    g = DeviceGraph.from_edges(V, src, dst, device=cuda)
    dims = [40, 16, 16]
    model = MoNet(g, dims, K, r, seed=4)
    snap = [(np64(Wc), np64(mu), np64(si), f) for Wc, mu, si, f in model.layers]
    H = feats(V, 40, cuda)
    loss, grads = model.train_step(H, lr=0.0)
    torch.cuda.synchronize()
    hg = O.host_graph(V, src, dst)
    xs, fws = [np64(H)], []
    views = lambda Wc, f: (Wc[:, :K * f], Wc[:, K * f:K * f + r], Wc[:, K * f + r:K * f + 2 * r])  # noqa: E731
    for Wc, mu, si, f in snap:
        fw = O.gmm_layer_fwd_f64(hg, xs[-1], *views(Wc, f), mu, si, K, r, f)
        fws.append(fw)
        xs.append(fw["out"])
    assert abs(float(loss.item()) - xs[-1].sum()) <= 1e-4 * max(1.0, abs(xs[-1].sum()))
    gr = np.ones_like(xs[-1])
    for i in reversed(range(len(snap))):
        Wc, mu, si, f = snap[i]
        bw = O.gmm_layer_bwd_f64(hg, xs[i], *views(Wc, f), mu, si, K, r, f, fws[i], gr, need_dH=i > 0)
        dW, dPl, dPr, dmu, dsinv = (np64(t) for t in grads[i][:5])
        for a, b in ((dW, bw["dW"]), (dPl, bw["dPl"]), (dPr, bw["dPr"]), (dmu, bw["dmu"]), (dsinv, bw["dsinv"])):
            assert norm_err(a, b) < 1e-4
        gr = bw["dH"]


def test_gcn_step_matches_oracle(cuda):
    V, E = 4000, 60000
    src, dst = uniform_edges(V, E, seed=6)
    g = DeviceGraph.from_edges(V, src, dst, device=cuda)
    dims = [32, 24, 24]
    model = GCN(g, dims, seed=7)
    snap = [(np64(W), np64(b)) for W, b in model.layers]
    H = feats(V, 32, cuda)
    loss, grads = model.train_step(H, lr=0.0)
    torch.cuda.synchronize()
    hg = O.host_graph(V, src, dst)
    w = O.gcn_norm(hg)
    xs, fws = [np64(H)], []
    for W, b in snap:
        fw = O.gcn_layer_fwd_f64(hg, xs[-1], W, b.reshape(-1), w)
        fws.append(fw)
        xs.append(fw["out"])
    assert abs(float(loss.item()) - xs[-1].sum()) <= 1e-4 * max(1.0, abs(xs[-1].sum()))
    gr = np.ones_like(xs[-1])
    for i in reversed(range(len(snap))):
        W, b = snap[i]
        bw = O.gcn_layer_bwd_f64(hg, xs[i], W, fws[i], gr, w)
        dW, db = (np64(t) for t in grads[i])
        assert norm_err(dW, bw["dW"]) < 1e-4 and norm_err(db.reshape(-1), bw["db"]) < 1e-4
        gr = bw["dH"]


@pytest.mark.parametrize("which", ["edgeconv", "monet"])
def test_graphed_step_replays_the_eager_step(cuda, which):
    """The CUDA-graph replay the bench uses for the launch-bound configs runs the same kernels:
    with lr = 0 the replayed loss equals the eager one bitwise."""
    if which == "edgeconv":
        src, dst = knn_edges(2, 256, 10, seed=1)
        g = DeviceGraph.from_edges(512, src, dst, device=cuda)
        model, H = EdgeConvNet(g, [16, 32, 32], seed=2), feats(512, 16, cuda)
    else:
        src, dst = uniform_edges(3000, 20000, seed=3)
        g = DeviceGraph.from_edges(3000, src, dst, device=cuda)
        model, H = MoNet(g, [40, 16, 16], 3, 3, seed=4), feats(3000, 40, cuda)
    eager = float(model.train_step(H, lr=0.0)[0].item())
    gs = GraphedStep(model, H, 0.0, warmup=1)
    gs.replay()
    torch.cuda.synchronize()
    assert float(gs.loss.item()) == eager and gs.kernels > 0
