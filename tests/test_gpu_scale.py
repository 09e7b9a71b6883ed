"""GPU: parity at the benchmarked scales, through the benchmarked model path.

Every test builds the graph with the bench's own generator and runs models.GAT -- the
bench's step: K1 tcgen05 transform with the LP epilogue, the lean K2 / K4f kernels, the
default edge-balance chunk (2048) and the work-counter item fetch (these graphs have far
more than 8 items per warp, so gnncg_gat_* attach the counter; K4f takes one item per
request at C2 and ~5 at the 100-edge-per-row graphs).  Bound 1e-4 (north_star) against f64:
  * forward outputs: the reference's elementwise rel_err = |a-b| / max(1,|a|,|b|)
    (tensor.hpp:153-156);
  * gradients: max-normalised |a-b| / max(1, max|ref|) -- the stated deviation of DESIGN.md
    §2.  They are sums over 10^5..10^9 fp32 terms; where entries cancel to near zero the
    elementwise bound is out of reach of ANY fp32 evaluation: the reference's own f32 CPU
    port, run on the same graph, measures elementwise 6.4e-3 on dW of layer 1 at C2
    (profiles/r02_c2_grad_conditioning.txt).  The elementwise errors of both are printed.
The graphs:
  * C2 (Reddit-shaped, 233K / 114M): the full 2-layer forward and every parameter gradient
    against the f64 OpenMP oracle (oracle.cpp gat_layer_*_omp<double>) on the same graph;
  * a 10M-edge graph from the C5 generator (100K vertices, mean degree 100, 3 layers of
    8 x 16): everything, the same way;
  * C5 itself (10M / 1B): sampled rows of the first and last layer outputs and of the last
    layer's input gradient against the f64 local-neighbourhood restatement (oracle/sampled.py),
    since a full CPU oracle would need minutes and ~100 GB.
"""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from oracle import sampled as S
from paper_2110_09524_b200.graph import DeviceGraph
from paper_2110_09524_b200.models import GAT

pytestmark = pytest.mark.gpu
BOUND = 1e-4


def features(V, fin, dev, seed=1234):
    gen = torch.Generator(device=dev)
    gen.manual_seed(seed)
    ld = (fin + 3) // 4 * 4
    return torch.rand(V, ld, generator=gen, device=dev).mul_(2).sub_(1)[:, :fin]


def host_graph(g: DeviceGraph) -> "O.HostGraph":
    h = g.to_host()
    return O.HostGraph(g.num_vertices, h["src"], h["dst"], h["dst_off"], h["dst_src"], h["dst_eid"], h["src_off"],
                       h["src_dst"], h["src_eid"])


def np64(t):
    return t.detach().double().cpu().numpy()


def full_parity(g, dims, dev):
    """One fwd + bwd of models.GAT (loss = sum of exits) against the f64 OpenMP oracle."""
    model = GAT(g, dims, seed=1)
    H = features(g.num_vertices, dims[0][0], dev)
    xs, stashes = model.forward(H)
    grads = model.backward(xs, stashes, model.seed_grad(xs[-1]))
    torch.cuda.synchronize()
    hg = host_graph(g)
    Hh = np64(H)
    fws, ins = [], [Hh]
    for L in model.layers:
        fw = O.gat_layer_fwd_omp(hg, ins[-1], np64(L.W), np64(L.a_l), np64(L.a_r), L.p.heads, L.p.f)
        fws.append(fw)
        ins.append(fw["out"])
    fwd, grads_norm, grads_elem = {}, {}, {}
    for i in range(len(model.layers)):
        fwd[f"out{i + 1}"] = O.max_rel_err(np64(xs[i + 1]), fws[i]["out"])
    grad = np.ones_like(ins[-1])
    for i in reversed(range(len(model.layers))):
        L = model.layers[i]
        bw = O.gat_layer_bwd_omp(hg, ins[i], np64(L.W), np64(L.a_l), np64(L.a_r), L.p.heads, L.p.f, fws[i], grad,
                                 need_dH=i > 0)
        gr = grads[i]
        pairs = [(f"dW{i + 1}", gr.dW, bw["dW"]), (f"da_l{i + 1}", gr.da_l, bw["dal"]),
                 (f"da_r{i + 1}", gr.da_r, bw["dar"])]
        if i > 0:
            pairs.append((f"dH{i + 1}", gr.dH, bw["dH"]))
        for name, got, ref in pairs:
            grads_norm[name] = S.max_norm_err(np64(got), ref)
            grads_elem[name] = O.max_rel_err(np64(got), ref)
        grad = bw["dH"]
    return fwd, grads_norm, grads_elem


def check(fwd, gnorm, gelem, tag):
    print(f"{tag} forward elementwise rel_err:", {k: f"{v:.2e}" for k, v in fwd.items()})
    print(f"{tag} gradients max-normalised:", {k: f"{v:.2e}" for k, v in gnorm.items()})
    print(f"{tag} gradients elementwise (reported):", {k: f"{v:.2e}" for k, v in gelem.items()})
    assert all(e < BOUND for e in fwd.values()), fwd
    assert all(e < BOUND for e in gnorm.values()), gnorm


def test_c2_reddit_full_forward_and_all_gradients(cuda):
    g = DeviceGraph.chung_lu(233_000, 114_000_000, offset=1100, seed=0, device=cuda)
    check(*full_parity(g, [(602, 8, 32), (256, 8, 32)], cuda), "C2")


def test_10m_edge_graph_full_parity(cuda):
    g = DeviceGraph.chung_lu(100_000, 10_000_000, offset=100, seed=0, device=cuda)
    check(*full_parity(g, [(128, 8, 16)] * 3, cuda), "10M-edge")


def test_c5_1b_edges_sampled_rows(cuda):
    g = DeviceGraph.chung_lu(10_000_000, 1_000_000_000, offset=10_000, seed=0, device=cuda)
    model = GAT(g, [(128, 8, 16)] * 3, seed=1)
    H = features(g.num_vertices, 128, cuda)
    res = S.gat_model_sampled_check(model, H, n_rows=16, n_src=3, seed=0, hub_src=False)
    print("C5 sampled:", res)
    assert res["max_in_degree_checked"] > 5000  # the hub rows (split into 2048-edge chunks) are among them
    assert res["max_rel_err"]["out_layer1"] < BOUND and res["max_rel_err"]["out_last"] < BOUND, res
    assert res["max_norm_err"]["dH_last"] < BOUND, res
