"""Operator IR, the three optimisation passes, and lowering onto the B200 kernels.

SURVEY §8(f) rank 4: "IR + passes (reorganize / plan_fusion / plan_recompute) driving the
kernels".  The reference specifies these modules but ships no code for them (
`src/ir.cpp`, `src/passes.cpp` are absent, `proj/CMakeLists.txt:21-22`).  This is a compact
restatement over the four paper models whose end product is a *kernel plan*: the list of
sm_100a kernels (libgnncg_b200.so) that execute the optimised graph.  Nothing here computes
tensor values; `compile_model(...).model(g)` hands back the runnable model built on exactly the
kernels the plan names.

  ir          OpNode / IRGraph, build_model (gcn | gat | edgeconv | monet),
              decompose, pretty printer
  passes      reorganize, plan_fusion (skew threshold 32 at
              SPEC.md:302), plan_recompute (op-count threshold 4 at SPEC.md:303)
  lowering    fused regions / expensive Applies -> B200 kernels
"""
from __future__ import annotations

from dataclasses import dataclass, field

SCATTER, GATHER, APPLY_EDGE, APPLY_VERTEX, AGGREGATE, REDUCE_SCATTER = (
    "Scatter", "Gather", "ApplyEdge", "ApplyVertex", "Aggregate", "ReduceScatter")
GRAPH_KINDS = (SCATTER, GATHER, AGGREGATE, REDUCE_SCATTER)
# linear vertex-applicable functions distribute over {add, sub, copy} scatters (SPEC.md:300 static
# table); an edge-weight product (mul_e) is linear too but needs the edge, so it stays edge-side
LINEAR_PREFIXES = ("lp:", "matmul:")
DISTRIBUTIVE_SCATTERS = ("u_add_v", "u_sub_v", "copy_u", "copy_v")
SKEW_THRESHOLD = 32
RECOMPUTE_MAX_OPS = 4


class IRError(ValueError):
    pass


class LoweringError(IRError):
    """A fused region that no B200 kernel implements (e.g. an un-reorganized GAT head)."""


@dataclass(frozen=True)
class OpNode:
    """SPEC.md:161-167.  `fn` is the phi / psi / apply-function tag; inputs are node ids or
    entry names; cost = expensive iff the apply contains a dense matmul."""

    id: int
    kind: str
    fn: str
    inputs: tuple
    out_class: str  # "vertex" | "edge"
    cost: str = "lightweight"

    def line(self) -> str:
        ins = ", ".join(str(i) for i in self.inputs)
        return f"{self.id}: {self.kind}[{self.fn}] ({ins}) -> {self.out_class}"


@dataclass
class IRGraph:
    model: str
    nodes: list = field(default_factory=list)
    entries: tuple = ("H",)
    exits: tuple = ()

    def add(self, kind, fn, inputs, out_class=None, cost="lightweight") -> int:
        if out_class is None:
            out_class = {SCATTER: "edge", GATHER: "vertex", AGGREGATE: "vertex", REDUCE_SCATTER: "edge"}.get(kind)
            if out_class is None:  # Apply-: graph-irrelevant, keeps its input's class
                out_class = self._class_of(inputs[0])
        n = OpNode(len(self.nodes), kind, fn, tuple(inputs), out_class, cost)
        self.nodes.append(n)
        return n.id

    def _class_of(self, ref) -> str:
        return "vertex" if isinstance(ref, str) else self.nodes[ref].out_class

    def node(self, i: int) -> OpNode:
        return self.nodes[i]

    def pretty(self) -> str:
        """One node per line, "id: Kind[fn] (inputs) -> class"."""
        return "\n".join(n.line() for n in self.nodes)

    def kinds(self) -> list:
        return [n.kind for n in self.nodes]

    def consumers(self, i: int) -> list:
        return [n.id for n in self.nodes if i in n.inputs]


# ----------------------------------------------------------------------------- builders
def build_model(model: str, heads: int = 1) -> IRGraph:
    """The unoptimised ("naive") layer of each paper model (App. A.2)."""
    g = IRGraph(model)
    if model == "gcn":  # [ApplyVertex(W), Scatter(copy_u), ApplyEdge(x e_uv), Gather(sum), ApplyVertex(+b, sigma)]
        x = g.add(APPLY_VERTEX, "matmul:W", ("H",), cost="expensive")
        e = g.add(SCATTER, "copy_u", (x,))
        e = g.add(APPLY_EDGE, "mul_e", (e,))
        v = g.add(GATHER, "sum", (e,))
        g.add(APPLY_VERTEX, "bias_relu", (v,))
    elif model == "gat":  # ApplyVertex(W) -> Scatter(u_concat_v) -> ApplyEdge(LP a, LeakyReLU) -> softmax -> Aggregate
        x = g.add(APPLY_VERTEX, "matmul:W", ("H",), cost="expensive")
        e = g.add(SCATTER, "u_concat_v", (x,))
        e = g.add(APPLY_EDGE, "lp:a", (e,), cost="expensive")  # per-edge LP over 2f values
        e = g.add(APPLY_EDGE, "leaky_relu", (e,))
        e = g.add(REDUCE_SCATTER, "edge_softmax", (e,))
        g.add(AGGREGATE, "sum_mul_u", (e, x))
    elif model == "edgeconv":  # [Scatter(u_sub_v), ApplyEdge(Theta), ApplyVertex(Phi), ApplyEdge(e_add_v), Gather(max)]
        e = g.add(SCATTER, "u_sub_v", ("H",))
        e = g.add(APPLY_EDGE, "matmul:Theta", (e,), cost="expensive")
        p = g.add(APPLY_VERTEX, "matmul:Phi", ("H",), cost="expensive")
        e = g.add(APPLY_EDGE, "e_add_v", (e, p))
        g.add(GATHER, "max", (e,))
    elif model == "monet":  # pseudo-coordinates of (x_u, x_v), K gaussian kernels, weighted sum
        x = g.add(APPLY_VERTEX, "matmul:W", ("H",), cost="expensive")
        e = g.add(SCATTER, "u_concat_v", ("H",))
        e = g.add(APPLY_EDGE, "lp:P", (e,), cost="expensive")
        e = g.add(APPLY_EDGE, "gaussian", (e,))
        g.add(AGGREGATE, "sum_mul_u", (e, x))
    else:
        raise IRError(f"unsupported model {model!r}")  # SPEC.md:184 errors
    g.exits = (len(g.nodes) - 1,)
    return g


# ----------------------------------------------------------------------------- decompose
def decompose(ir: IRGraph) -> IRGraph:
    """Aggregate -> Scatter, ApplyEdge, Gather; ReduceScatter(edge_softmax) -> the RS1/RS2 chain
    (PAPER.md:527-530).  Idempotent; identity without composites."""
    out = IRGraph(ir.model, entries=ir.entries)
    remap = {}

    def m(ref):
        return ref if isinstance(ref, str) else remap[ref]

    for n in ir.nodes:
        ins = tuple(m(i) for i in n.inputs)
        if n.kind == AGGREGATE:  # (edge weights, vertex features)
            w, x = ins
            s = out.add(SCATTER, "copy_u", (x,))
            a = out.add(APPLY_EDGE, "mul", (s, w))
            remap[n.id] = out.add(GATHER, "sum", (a,))
        elif n.kind == REDUCE_SCATTER:
            (z,) = ins
            mx = out.add(GATHER, "max", (z,))
            s = out.add(SCATTER, "copy_v", (mx,))
            d = out.add(APPLY_EDGE, "sub", (z, s))
            ex = out.add(APPLY_EDGE, "exp", (d,))
            sm = out.add(GATHER, "sum", (ex,))
            s2 = out.add(SCATTER, "copy_v", (sm,))
            remap[n.id] = out.add(APPLY_EDGE, "div", (ex, s2))
        else:
            remap[n.id] = out.add(n.kind, n.fn, ins, n.out_class, n.cost)
    out.exits = tuple(remap[e] for e in ir.exits)
    return out


# ----------------------------------------------------------------------------- reorganize
def _is_linear(fn: str) -> bool:
    return fn.startswith(LINEAR_PREFIXES)


def reorganize(ir: IRGraph) -> IRGraph:
    """Postpone Scatter past linear ApplyEdge (§4):
      Scatter(phi in {add, sub, copy}) -> ApplyEdge(linear f)   =>  ApplyVertex(f) -> Scatter(phi)
      Scatter(u_concat_v) -> ApplyEdge(LP a)  =>  ApplyVertex(a_l), ApplyVertex(a_r) -> Scatter(u_add_v)
    Non-distributive pairs (LeakyReLU, exp, ...) are left untouched.  Total and semantics
    preserving; a no-op when nothing matches."""
    out = IRGraph(ir.model, entries=ir.entries)
    remap, skip = {}, set()

    def m(ref):
        return ref if isinstance(ref, str) else remap[ref]

    for n in ir.nodes:
        if n.id in skip:
            continue
        cons = ir.consumers(n.id)
        nxt = ir.node(cons[0]) if len(cons) == 1 else None
        if n.kind == SCATTER and nxt is not None and nxt.kind == APPLY_EDGE and len(nxt.inputs) == 1:
            src = tuple(m(i) for i in n.inputs)
            if n.fn == "u_concat_v" and nxt.fn.startswith("lp:"):
                name = nxt.fn[3:]
                al = out.add(APPLY_VERTEX, f"lp:{name}_l", src, "vertex")
                ar = out.add(APPLY_VERTEX, f"lp:{name}_r", src, "vertex")
                remap[nxt.id] = out.add(SCATTER, "u_add_v", (al, ar))
                skip.add(nxt.id)
                continue
            if n.fn in DISTRIBUTIVE_SCATTERS and _is_linear(nxt.fn):
                v = out.add(APPLY_VERTEX, nxt.fn, src, "vertex", nxt.cost)
                remap[nxt.id] = out.add(SCATTER, n.fn, (v,))
                skip.add(nxt.id)
                continue
        remap[n.id] = out.add(n.kind, n.fn, tuple(m(i) for i in n.inputs), n.out_class, n.cost)
    out.exits = tuple(remap[e] for e in ir.exits)
    return out


def hoist_vertex_side(ir: IRGraph) -> IRGraph:
    """Stable topological reorder: every node that depends on no graph operator (the hoisted
    vertex-side Applies) comes first, so the graph operators form one contiguous chain and
    fusion regions are not cut by an independent barrier (reorganize first, so
    barriers moved vertex-side maximise region size)."""
    dep = {}
    for n in ir.nodes:
        dep[n.id] = n.kind in GRAPH_KINDS or any(dep.get(i, False) for i in n.inputs if not isinstance(i, str))
    order = [n for n in ir.nodes if not dep[n.id]] + [n for n in ir.nodes if dep[n.id]]
    out = IRGraph(ir.model, entries=ir.entries)
    remap = {}
    for n in order:
        remap[n.id] = out.add(n.kind, n.fn, tuple(i if isinstance(i, str) else remap[i] for i in n.inputs),
                              n.out_class, n.cost)
    out.exits = tuple(remap[e] for e in ir.exits)
    return out


# ----------------------------------------------------------------------------- plan_fusion
@dataclass
class Region:
    members: tuple
    mapping: str  # "vertex_balanced" | "edge_balanced"


@dataclass
class FusionPlan:
    regions: list
    barriers: tuple  # expensive Apply nodes, never inside a region


def _reduce_scatter_shaped(ir: IRGraph, members) -> bool:
    """A Gather whose result feeds a Scatter inside the region (the edge-softmax shape)."""
    ms = set(members)
    return any(ir.node(i).kind == GATHER and any(ir.node(c).kind == SCATTER for c in ir.consumers(i) if c in ms)
               for i in members)


def plan_fusion(ir: IRGraph, max_in_degree: int = 1, mean_in_degree: float = 1.0, override: str | None = None):
    """Maximal contiguous runs of graph-related ops and lightweight Applies, split at expensive
    Applies.  Mapping: forced vertex_balanced on ReduceScatter-shaped regions
    (an online-softmax merge would be needed otherwise); else edge_balanced when
    max_in / max(1, mean_in) > 32; `override` wins when legal."""
    regions, cur, barriers = [], [], []

    def close():
        if cur and any(ir.node(i).kind in GRAPH_KINDS for i in cur):
            forced = _reduce_scatter_shaped(ir, cur)
            mapping = "edge_balanced" if max_in_degree / max(1.0, mean_in_degree) > SKEW_THRESHOLD else "vertex_balanced"
            if forced:
                mapping = "vertex_balanced"
            if override is not None:
                if forced and override == "edge_balanced":
                    raise IRError("plan_fusion: edge_balanced is illegal on a ReduceScatter region (SPEC.md:268)")
                mapping = override
            regions.append(Region(tuple(cur), mapping))
        cur.clear()

    for n in ir.nodes:
        if n.cost == "expensive":
            close()
            barriers.append(n.id)
        elif n.kind in GRAPH_KINDS or cur:
            cur.append(n.id)
        # lightweight vertex Applies before any graph op stay outside (vertex-side work)
    close()
    return FusionPlan(regions, tuple(barriers))


# ----------------------------------------------------------------------------- plan_recompute
def plan_recompute(ir: IRGraph, fusion: FusionPlan) -> dict:
    """Per region-internal tensor: O(|V|) (vertex class) -> "stash"; O(|E|) (edge class) ->
    "recompute" when its producing chain inside the region is lightweight and at most
    RECOMPUTE_MAX_OPS long, else "stash"."""
    labels = {}
    for reg in fusion.regions:
        ms = set(reg.members)
        for i in reg.members:
            n = ir.node(i)
            if n.out_class == "vertex":
                labels[i] = "stash"
                continue
            depth, frontier, ok = 0, [i], True
            while frontier and ok:
                nxt = []
                for j in frontier:
                    node = ir.node(j)
                    if node.cost == "expensive":
                        ok = False
                    if node.kind != GATHER:  # a Gather output is a stashed O(|V|) leaf
                        nxt += [k for k in node.inputs if not isinstance(k, str) and k in ms]
                depth += 1
                frontier = nxt
                if depth > RECOMPUTE_MAX_OPS * 2:
                    ok = False
            labels[i] = "recompute" if ok else "stash"
    return labels


# ----------------------------------------------------------------------------- lowering
@dataclass
class KernelPlan:
    model: str
    kernels: list  # (kernel name, node ids it implements)

    def names(self) -> list:
        return [k for k, _ in self.kernels]


def _region_signature(ir: IRGraph, reg: Region) -> tuple:
    return tuple(f"{ir.node(i).kind}[{ir.node(i).fn}]" for i in reg.members)


_REGION_KERNELS = {
    # reorganized + decomposed GAT region: Scatter(u_add_v), LeakyReLU, RS1/RS2 edge-softmax, Aggregate
    "gat": ("gnncg_gat_fwd / gnncg_gat_bwd_src_fused (K2 / K4f)",
            ("Scatter[u_add_v]", "ApplyEdge[leaky_relu]", "Gather[max]", "Scatter[copy_v]", "ApplyEdge[sub]",
             "ApplyEdge[exp]", "Gather[sum]", "Scatter[copy_v]", "ApplyEdge[div]", "Scatter[copy_u]",
             "ApplyEdge[mul]", "Gather[sum]")),
    "edgeconv": ("gnncg_edgeconv_fwd / gnncg_edgeconv_bwd (K6 / K7)",
                 ("Scatter[u_sub_v]", "ApplyEdge[e_add_v]", "Gather[max]")),
    "gcn": ("gnncg_spmm (weighted aggregate, fused bias + ReLU)",
            ("Scatter[copy_u]", "ApplyEdge[mul_e]", "Gather[sum]", "ApplyVertex[bias_relu]")),
    "monet": ("gnncg_gmm_fwd / gnncg_gmm_bwd (K8)",
              ("Scatter[u_add_v]", "ApplyEdge[gaussian]", "Scatter[copy_u]", "ApplyEdge[mul]", "Gather[sum]")),
}


def lower(ir: IRGraph, fusion: FusionPlan) -> KernelPlan:
    """Map the planned graph onto libgnncg_b200 kernels.  Both mappings of a region lower to the
    same kernel, whose work items are destination (or source) rows with hub rows split into
    edge chunks merged in a fixed order -- the spec's two schemes in one schedule.
    Expensive ApplyVertex -> the tcgen05
    GEMM (the GAT LPs that follow it ride in its epilogue, gnncg_gat_transform); each fused region
    -> the one kernel that implements exactly that region.  A region no kernel implements (the
    naive GAT with a per-edge LP, an un-reorganized EdgeConv) is a LoweringError: the B200 build
    has no generic per-operator fallback."""
    kernels = []
    lp_nodes = [n.id for n in ir.nodes if n.kind == APPLY_VERTEX and n.fn.startswith("lp:")]
    for b in fusion.barriers:
        n = ir.node(b)
        if n.kind != APPLY_VERTEX or not n.fn.startswith("matmul:"):
            raise LoweringError(f"no B200 kernel for expensive {n.kind}[{n.fn}] (per-edge dense work)")
        epi = [i for i in lp_nodes if ir.node(i).inputs == (b,)]          # LPs of its output
        cols = [i for i in lp_nodes if ir.node(i).inputs == n.inputs]      # LPs of its input
        if epi:
            kernels.append(("gnncg_gat_transform (tcgen05 GEMM + LP epilogue)", (b, *epi)))
        elif cols:
            kernels.append(("gnncg_gemm (tcgen05 3xTF32, projections as extra columns)", (b, *cols)))
        else:
            kernels.append(("gnncg_gemm (tcgen05 3xTF32)", (b,)))
    for reg in fusion.regions:
        sig = _region_signature(ir, reg)
        spec = _REGION_KERNELS.get(ir.model)
        if spec is None or sig != spec[1]:
            raise LoweringError(f"no B200 kernel implements region {list(sig)} ({reg.mapping})")
        kernels.append((spec[0], reg.members))
    return KernelPlan(ir.model, kernels)


@dataclass
class Compiled:
    """compile_model's result: the optimised IR, its plans, and the kernel plan."""

    naive: IRGraph
    ir: IRGraph
    fusion: FusionPlan
    recompute: dict
    plan: KernelPlan

    def model(self, g, dims, **kw):
        """The runnable model on exactly the kernels of `plan` (paper_2110_09524_b200.models)."""
        from . import models

        cls = {"gat": models.GAT, "edgeconv": models.EdgeConvNet, "monet": models.MoNet, "gcn": models.GCN}
        return cls[self.ir.model](g, dims, **kw)


def compile_model(model: str, max_in_degree: int = 1, mean_in_degree: float = 1.0, opt: str = "all") -> Compiled:
    """build_model -> reorganize -> decompose -> plan_fusion -> plan_recompute -> lower
    (the spec's pipeline order, SPEC.md:148 note: reorganize before fusion).  opt = "none" skips
    the reorganization (and then fails to lower for GAT / MoNet / EdgeConv: the naive forms
    carry per-edge dense work)."""
    naive = build_model(model)
    ir = reorganize(naive) if opt != "none" else naive
    ir = hoist_vertex_side(decompose(ir))
    fusion = plan_fusion(ir, max_in_degree, mean_in_degree)
    return Compiled(naive, ir, fusion, plan_recompute(ir, fusion), lower(ir, fusion))
