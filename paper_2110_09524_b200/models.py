"""Layer stacks and the training step (train_step) over the fused ops.

``GAT`` is the benchmark model: L GAT layers, identity between layers (the paper's
GAT layer ends at the aggregation; the spec's "-> (next layer)",
SPEC.md:181 -- recorded in DESIGN.md), loss = sum of the exit tensor
(seed gradient all ones), SGD update params -= lr * grad.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _lib
from ._lib import call
from .graph import DeviceGraph, _ptr, _stream
from .ops import GatParams, gat_backward, gat_forward


def init_uniform(rows: int, cols: int, gen: torch.Generator, device) -> torch.Tensor:
    """U(-s, s) with s = 1/sqrt(cols) -- the scale of init_seeded (tensor.hpp:44-63)."""
    s = 1.0 / (cols ** 0.5) if cols else 0.0
    t = torch.rand(rows, cols, generator=gen, device=device, dtype=torch.float32)
    return t.mul_(2 * s).sub_(s)


@dataclass
class GatLayerParams:
    W: torch.Tensor
    a_l: torch.Tensor
    a_r: torch.Tensor
    p: GatParams


class GAT:
    """A stack of GAT layers: dims = [(F_in, heads, f), ...]; layer l+1 has F_in = heads*f of layer l."""

    def __init__(self, g: DeviceGraph, dims, seed: int = 0, slope: float = 0.2, chunk: int | None = None,
                 mode: str = "auto"):
        self.g = g
        self.chunk = chunk
        self.mode = mode  # backward: "auto" (fast when supported) | "fast" | "deterministic"
        dev = g.device
        gen = torch.Generator(device=dev)
        gen.manual_seed(seed)
        self.layers: list[GatLayerParams] = []
        for fin, h, f in dims:
            self.layers.append(GatLayerParams(init_uniform(fin, h * f, gen, dev), init_uniform(h, f, gen, dev),
                                              init_uniform(h, f, gen, dev), GatParams(h, f, slope)))
        self.loss = torch.zeros(4, device=dev)  # [0] = loss; padded for alignment
        self._sum_ws = torch.empty(_lib.lib().gnncg_sum_workspace(), dtype=torch.uint8, device=dev)
        self._ones = None

    def forward(self, H: torch.Tensor):
        xs, stashes = [H], []
        for L in self.layers:
            out, st = gat_forward(self.g, xs[-1], L.W, L.a_l, L.a_r, L.p, chunk=self.chunk)
            xs.append(out)
            stashes.append(st)
        return xs, stashes

    def backward(self, xs, stashes, dOut: torch.Tensor):
        grads = [None] * len(self.layers)
        g = dOut
        for i in reversed(range(len(self.layers))):
            L = self.layers[i]
            gr = gat_backward(self.g, xs[i], L.W, L.a_l, L.a_r, stashes[i], g, L.p, need_dH=i > 0, chunk=self.chunk,
                              mode=self.mode)
            grads[i] = gr
            g = gr.dH
        return grads

    def seed_grad(self, like: torch.Tensor) -> torch.Tensor:
        """dLoss/dOut for loss = sum(out): all ones, filled on the device."""
        if self._ones is None or self._ones.shape != like.shape:
            self._ones = torch.empty_like(like)
            call("gnncg_fill", self._ones.numel(), 1.0, _ptr(self._ones), _stream())
        return self._ones

    def sgd(self, grads, lr: float):
        s = _stream()
        for L, gr in zip(self.layers, grads):
            for p, dp in ((L.W, gr.dW), (L.a_l, gr.da_l), (L.a_r, gr.da_r)):
                call("gnncg_sgd_update", p.numel(), lr, _ptr(dp), _ptr(p), s)

    def train_step(self, H: torch.Tensor, lr: float = 0.0, dOut: torch.Tensor | None = None):
        """forward -> loss -> backward -> params -= lr * grad.  Returns (loss tensor (device), grads)."""
        xs, stashes = self.forward(H)
        out = xs[-1]
        call("gnncg_sum", out.numel(), _ptr(out), _ptr(self.loss), _ptr(self._sum_ws), self._sum_ws.numel(),
             _stream())
        grads = self.backward(xs, stashes, self.seed_grad(out) if dOut is None else dOut)
        self.sgd(grads, lr)
        return self.loss[:1], grads
