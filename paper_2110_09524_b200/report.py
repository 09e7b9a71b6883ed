"""Cost report of a GAT layer on the B200 path (the reference's `compare` JSON):
one forward + fused backward through the product kernels with the device cost counters on,
checked against the closed forms of cost.py, plus the modelled opt levels."""
from __future__ import annotations

import torch

from . import _lib, cost
from .graph import DeviceGraph, _ptr
from .ops import GatParams, GatStash, fast_supported, gat_region_backward, gat_region_forward, gat_transform

NUM_COUNTERS = 10


class CostCounters:
    """Context manager: gnncg_cost_counters on a zeroed device array for the duration."""

    def __init__(self, device):
        self.buf = torch.zeros(NUM_COUNTERS, dtype=torch.int64, device=device)

    def __enter__(self):
        torch.cuda.synchronize()
        _lib.call("gnncg_cost_counters", _ptr(self.buf))
        return self

    def __exit__(self, *exc):
        torch.cuda.synchronize()
        _lib.call("gnncg_cost_counters", None)

    def values(self):
        return self.buf.cpu().tolist()


def gat_layer_report(g: DeviceGraph, H: torch.Tensor, W, a_l, a_r, p: GatParams, dOut=None, config=None) -> dict:
    """Run one GAT layer forward + fused backward with the counters on and return the compare
    report (cost.compare_report) for it."""
    V, E, h, f = g.num_vertices, g.num_edges, p.heads, p.f
    dev = H.device
    dOut = torch.ones(V, h * f, device=dev) if dOut is None else dOut
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    resident = torch.cuda.memory_allocated()
    torch.cuda.reset_peak_memory_stats()
    with CostCounters(dev) as cc:
        s.record()
        Ht, Al, Ar = gat_transform(H, W, a_l, a_r, h, f, ws=g.ws)
        out, m, d = gat_region_forward(g, Ht, Al, Ar, p)
        e.record()
        fast = fast_supported(p)
        gat_region_backward(g, GatStash(Ht, Al, Ar, m, d, out), a_l, a_r, dOut, p,
                            mode="fast" if fast else "deterministic")
    peak = torch.cuda.max_memory_allocated() - resident
    meas = cost.measured_from_counters(cc.values(), h, f)
    if not fast:  # K3 + K4 ran: the K4f io model does not apply
        meas["io_units"]["bwd"] = None
    mi, mean, _ = g.degree_stats()
    rep = cost.compare_report(V, E, h, f, {"max_in": int(mi), "mean_in": float(mean)}, measured=meas,
                              wall_ms=s.elapsed_time(e), peak_bytes=int(peak), config=config)
    rep["counters"] = {"edges": meas["edges"], "rows": meas["rows"], "lp_rows": meas["lp_rows"]}
    return rep
