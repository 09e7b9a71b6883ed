"""Closed-form cost algebra of the GAT layer (the reference's cost_model).

Element counts as the paper and spec define them, so they can be reported beside what
ncu measures:
  attention FLOPs   naive 6|E|f + |E|  -> reorganized 4|V|f + 2|E|      (per head)
  graph-op IO       unfused |V|hf + 7|E|h + 3|E|hf -> fused |V|hf + 5|E|h + 2|E|hf
  stash memory      fusion+stash keeps the O(|E| h) edge values (scores, weights) for the
                    backward; fusion+recompute keeps O(|V| h) (m, d) only
Known answers: G3 (|V| = |E| = 3), f = 2, h = 1 -> FLOPs 39 -> 30, IO 45 -> 33.
"""
from __future__ import annotations


def gat_attention_flops(V: int, E: int, f: int, h: int = 1) -> dict:
    return {"naive": h * (6 * E * f + E), "reorganized": h * (4 * V * f + 2 * E)}


def gat_io_units(V: int, E: int, h: int, f: int) -> dict:
    return {"unfused": V * h * f + 7 * E * h + 3 * E * h * f, "fused": V * h * f + 5 * E * h + 2 * E * h * f}


def gat_stash_units(V: int, E: int, h: int) -> dict:
    """Scalars kept from forward to backward by the fused region (excluding vertex inputs)."""
    return {"fusion_stash": 2 * E * h, "fusion_recompute": 2 * V * h}


def gat_layer_report(V: int, E: int, h: int, f: int, bytes_per_unit: int = 4) -> dict:
    fl = gat_attention_flops(V, E, f, h)
    io = gat_io_units(V, E, h, f)
    st = gat_stash_units(V, E, h)
    return {
        "attention_flops": fl, "flops_reduction": fl["naive"] / fl["reorganized"],
        "io_units": io, "io_reduction": io["unfused"] / io["fused"],
        "stash_units": st, "stash_bytes_saved": (st["fusion_stash"] - st["fusion_recompute"]) * bytes_per_unit,
    }


# ----------------------------------------------------------------------------- executed plan
# What the B200 kernels of the "all" plan (reorganize + fusion + recompute) do per GAT layer,
# as closed forms: the predictions that the device cost counters (gnncg_cost_counters) are
# checked against with integer equality.  Elements, index arrays excluded.
def gat_executed_flops(V: int, E: int, h: int, f: int) -> int:
    """Attention flops of the reorganized layer (PAPER.md:285 per head): the two vertex LPs in
    K1's epilogue (4 f per row and head) and u_add_v + LeakyReLU per edge and head in K2."""
    return 4 * V * f * h + 2 * E * h


def gat_executed_io(V: int, E: int, h: int, f: int) -> dict:
    """Boundary elements of the fused kernels.  K2 (forward region): per edge A_l[u] and the
    Ht[u] row are gathered; per destination row A_r is read and out, m, d written.  K4f (fused
    backward): per edge the destination record (A_r, lse, c per head) and the dOut[v] row are
    gathered and dz reduced into dA_r[v]; per source row Ht[u], A_l[u] are read and dHt, dA_l
    written."""
    hf = h * f
    return {"fwd": E * (h + hf) + V * (h + hf + 2 * h),
            "bwd": E * (3 * h + hf + h) + V * (2 * hf + 2 * h)}


COUNTER_SLOTS = {"K2": 0, "K3": 1, "K4": 2, "K4f": 3, "LP": 4}


def measured_from_counters(c, h: int, f: int) -> dict:
    """Flops / io units of one layer from the device counters (10 uint64: (edges, rows) pairs
    per kernel kind, COUNTER_SLOTS; the LP pair is (rows, calls))."""
    hf = h * f
    pair = {k: (int(c[2 * s]), int(c[2 * s + 1])) for k, s in COUNTER_SLOTS.items()}
    e2, r2 = pair["K2"]
    e4, r4 = pair["K4f"]
    return {"flops": 4 * f * h * pair["LP"][0] + 2 * h * e2,
            "io_units": {"fwd": e2 * (h + hf) + r2 * (h + hf + 2 * h), "bwd": e4 * (4 * h + hf) + r4 * (2 * hf + 2 * h)},
            "edges": {k: v[0] for k, v in pair.items() if k != "LP"}, "rows": {k: v[1] for k, v in pair.items()
                                                                                if k != "LP"},
            "lp_rows": pair["LP"][0]}


def compare_report(V: int, E: int, h: int, f: int, graph_stats: dict, measured: dict | None = None,
                   wall_ms: float | None = None, peak_bytes: int | None = None, config: dict | None = None) -> dict:
    """The reference's `compare` report (schema SPEC.md:466) for one GAT layer:
    the four opt levels of the cost model, with the executed level ("all") measured on the GPU.
    The other levels are modelled, not executed here (the B200 path runs the fused plan only)."""
    fl = gat_attention_flops(V, E, f, h)
    io = gat_io_units(V, E, h, f)
    st = gat_stash_units(V, E, h)
    hf = h * f
    # stash kept from forward to backward, in floats: the vertex inputs (Ht, A_l, A_r) plus the
    # edge-softmax state -- per edge (scores + weights) unless recomputed
    vert = V * (hf + 2 * h)
    results = [
        {"opt": "none", "mapping": "vertex_balanced", "flops": fl["naive"], "io_units": io["unfused"],
         "peak_mem_units": vert + st["fusion_stash"], "wall_ms": None, "checks": {"executed": False}},
        {"opt": "reorg", "mapping": "vertex_balanced", "flops": fl["reorganized"], "io_units": io["unfused"],
         "peak_mem_units": vert + st["fusion_stash"], "wall_ms": None, "checks": {"executed": False}},
        {"opt": "reorg+fusion", "mapping": "vertex_balanced", "flops": fl["reorganized"], "io_units": io["fused"],
         "peak_mem_units": vert + st["fusion_stash"], "wall_ms": None, "checks": {"executed": False}},
    ]
    pred_io = gat_executed_io(V, E, h, f)
    pred = {"flops": gat_executed_flops(V, E, h, f), "io_units": pred_io["fwd"]}
    allr = {"opt": "all", "mapping": "vertex_balanced (edge-balanced split rows, online-softmax merge)",
            "flops": pred["flops"], "io_units": pred["io_units"], "peak_mem_units": vert + st["fusion_recompute"],
            "wall_ms": wall_ms, "predicted": {**pred, "io_units_bwd": pred_io["bwd"]},
            "checks": {"executed": measured is not None}}
    if measured is not None:
        allr["measured"] = {"flops": measured["flops"], "io_units": measured["io_units"]["fwd"],
                            "io_units_bwd": measured["io_units"]["bwd"]}
        allr["flops"], allr["io_units"] = measured["flops"], measured["io_units"]["fwd"]
        allr["checks"].update({"flops_measured_eq_predicted": measured["flops"] == pred["flops"],
                               "io_measured_eq_predicted": measured["io_units"]["fwd"] == pred["io_units"]})
        if measured["io_units"]["bwd"] is not None:
            allr["checks"]["io_bwd_measured_eq_predicted"] = measured["io_units"]["bwd"] == pred_io["bwd"]
    if peak_bytes is not None:
        allr["peak_mem_units_measured"] = peak_bytes // 4
    results.append(allr)
    return {"version": 1, "config": config or {}, "graph": {"V": V, "E": E, **graph_stats}, "results": results}
