"""CPU: the operator IR, its passes and the lowering onto the B200 kernels
(paper_2110_09524_b200/ir.py) against the spec's examples."""
import pytest

from paper_2110_09524_b200 import ir as I


def seq(g):
    return [f"{n.kind}[{n.fn}]" for n in g.nodes]


def test_build_model_examples():
    # gcn, 1 layer
    assert seq(I.build_model("gcn")) == ["ApplyVertex[matmul:W]", "Scatter[copy_u]", "ApplyEdge[mul_e]", "Gather[sum]",
                                         "ApplyVertex[bias_relu]"]
    # edgeconv
    assert seq(I.build_model("edgeconv")) == ["Scatter[u_sub_v]", "ApplyEdge[matmul:Theta]", "ApplyVertex[matmul:Phi]",
                                              "ApplyEdge[e_add_v]", "Gather[max]"]
    # gat naive form: Scatter(u_concat_v) followed by an expensive ApplyEdge
    g = I.build_model("gat")
    i = next(n.id for n in g.nodes if n.fn == "u_concat_v")
    assert g.node(i + 1).kind == I.APPLY_EDGE and g.node(i + 1).cost == "expensive"
    with pytest.raises(I.IRError):
        I.build_model("transformer")


def test_output_classes_and_printer():
    g = I.build_model("gcn")
    assert [n.out_class for n in g.nodes] == ["vertex", "edge", "edge", "vertex", "vertex"]
    assert g.pretty().splitlines()[1] == "1: Scatter[copy_u] (0) -> edge"


def test_decompose_examples():
    g = I.decompose(I.build_model("gat"))
    s = seq(g)
    # Aggregate(sum, x m_e, copy_u) -> [Scatter(copy_u), ApplyEdge(mul), Gather(sum)]
    assert s[-3:] == ["Scatter[copy_u]", "ApplyEdge[mul]", "Gather[sum]"]
    # edge-softmax ReduceScatter -> RS1/RS2
    k = s.index("Gather[max]")
    assert s[k:k + 7] == ["Gather[max]", "Scatter[copy_v]", "ApplyEdge[sub]", "ApplyEdge[exp]", "Gather[sum]",
                          "Scatter[copy_v]", "ApplyEdge[div]"]
    # closure: only the four basic operators remain
    for m in ("gcn", "gat", "edgeconv", "monet"):
        assert set(I.decompose(I.build_model(m)).kinds()) <= {I.SCATTER, I.GATHER, I.APPLY_EDGE, I.APPLY_VERTEX}
    # idempotent, and the identity without composites
    assert I.decompose(g).pretty() == g.pretty()
    e = I.build_model("edgeconv")
    assert I.decompose(e).pretty() == e.pretty()


def test_reorganize_examples():
    # [Scatter(u_sub_v), ApplyEdge(LP Theta)] -> [ApplyVertex(LP Theta), Scatter(u_sub_v)]
    g = I.IRGraph("t")
    s = g.add(I.SCATTER, "u_sub_v", ("H",))
    g.add(I.APPLY_EDGE, "lp:Theta", (s,))
    g.exits = (1,)
    assert seq(I.reorganize(g)) == ["ApplyVertex[lp:Theta]", "Scatter[u_sub_v]"]
    # GAT attention head -> [ApplyVertex(a_l), ApplyVertex(a_r), Scatter(u_add_v), ApplyEdge(LeakyReLU)]
    r = seq(I.reorganize(I.build_model("gat")))
    k = r.index("ApplyVertex[lp:a_l]")
    assert r[k:k + 4] == ["ApplyVertex[lp:a_l]", "ApplyVertex[lp:a_r]", "Scatter[u_add_v]", "ApplyEdge[leaky_relu]"]
    assert "Scatter[u_concat_v]" not in r
    # [Scatter(u_sub_v), ApplyEdge(LeakyReLU)] -> unchanged (a nonlinearity blocks distribution)
    h = I.IRGraph("t")
    s = h.add(I.SCATTER, "u_sub_v", ("H",))
    h.add(I.APPLY_EDGE, "leaky_relu", (s,))
    h.exits = (1,)
    assert I.reorganize(h).pretty() == h.pretty()
    # the edge-weight product cannot move vertex-side
    assert seq(I.reorganize(I.build_model("gcn"))) == seq(I.build_model("gcn"))


def test_plan_fusion_examples():
    c = I.compile_model("gat", max_in_degree=20000, mean_in_degree=489)
    assert len(c.fusion.regions) == 1 and c.fusion.regions[0].mapping == "vertex_balanced"  # forced (RS shape)
    reg = c.fusion.regions[0]
    assert {c.ir.node(i).kind for i in reg.members} <= {I.SCATTER, I.GATHER, I.APPLY_EDGE}
    with pytest.raises(I.IRError):
        I.plan_fusion(c.ir, 20000, 489, override="edge_balanced")
    # EdgeConv: Theta and Phi are barriers, the graph ops fuse around them
    e = I.compile_model("edgeconv")
    assert [e.ir.node(b).fn for b in e.fusion.barriers] == ["matmul:Theta", "matmul:Phi"]
    assert len(e.fusion.regions) == 1
    # star(V=1000): max_in 999, mean 0.999 -> ratio 999 > 32 -> edge_balanced without RS shape
    assert I.compile_model("gcn", 999, 0.999).fusion.regions[0].mapping == "edge_balanced"
    assert I.compile_model("gcn", 10, 5.0).fusion.regions[0].mapping == "vertex_balanced"


def test_plan_recompute_examples():
    c = I.compile_model("gat")
    fn = {i: f"{c.ir.node(i).kind}[{c.ir.node(i).fn}]" for i in c.recompute}
    lab = {}
    for i, l in c.recompute.items():
        lab.setdefault(fn[i], set()).add(l)
    assert lab["Scatter[u_add_v]"] == {"recompute"}    # scatter_out
    assert lab["Gather[max]"] == {"stash"}             # softmax max, O(|V|)
    assert lab["ApplyEdge[div]"] == {"recompute"}      # edge weights
    k = [i for i in c.recompute if fn[i] == "Gather[sum]"][0]  # softmax denominator
    assert c.recompute[k] == "stash"
    e = I.compile_model("edgeconv")
    assert [l for i, l in e.recompute.items() if e.ir.node(i).kind == I.GATHER] == ["stash"]  # O(|V|) argmax side


def test_lowering_to_b200_kernels():
    names = {m: I.compile_model(m).plan.names() for m in ("gat", "edgeconv", "gcn", "monet")}
    assert names["gat"][0].startswith("gnncg_gat_transform") and "gnncg_gat_fwd" in names["gat"][1]
    assert sum(n.startswith("gnncg_gemm") for n in names["edgeconv"]) == 2 and "edgeconv" in names["edgeconv"][2]
    assert "spmm" in names["gcn"][1]
    assert "extra columns" in names["monet"][0] and "gmm" in names["monet"][1]
    # un-reorganized forms carry per-edge dense work: no kernel implements them (no CPU fallback)
    for m in ("gat", "edgeconv", "monet"):
        with pytest.raises(I.LoweringError):
            I.compile_model(m, opt="none")
