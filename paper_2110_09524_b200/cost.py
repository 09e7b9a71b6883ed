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
