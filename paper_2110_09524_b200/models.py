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
                 mode: str = "auto", gather: str = "fp32"):
        self.g = g
        self.chunk = chunk
        self.mode = mode  # backward: "auto" (fast when supported) | "fast" | "deterministic"
        self.gather = gather  # "fp32" | "bf16" gather tables (ops.GatParams)
        dev = g.device
        gen = torch.Generator(device=dev)
        gen.manual_seed(seed)
        self.layers: list[GatLayerParams] = []
        for fin, h, f in dims:
            self.layers.append(GatLayerParams(init_uniform(fin, h * f, gen, dev), init_uniform(h, f, gen, dev),
                                              init_uniform(h, f, gen, dev), GatParams(h, f, slope, gather)))
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


class EdgeConvNet:
    """EdgeConv stack (the paper's DGCNN setting uses layers {64,64,128,256},
    PAPER.md:409): dims = [F0, F1, ...]; layer l maps F_l -> F_{l+1}; identity between layers,
    loss = sum of exits, SGD.  Each layer's Theta and Phi are the two column halves of one
    parameter buffer [Theta | Phi], so the step runs on the library's kernels only (no
    concatenation or slicing copies)."""

    def __init__(self, g: DeviceGraph, dims, seed: int = 0):
        self.g = g
        dev = g.device
        gen = torch.Generator(device=dev)
        gen.manual_seed(seed)
        self.layers = []
        for a, b in zip(dims[:-1], dims[1:]):
            Th, Ph = init_uniform(a, b, gen, dev), init_uniform(a, b, gen, dev)
            Wcat = torch.cat([Th, Ph], dim=1)  # once, at init
            self.layers.append(Wcat)
        self.loss = torch.zeros(4, device=dev)
        self._sum_ws = torch.empty(_lib.lib().gnncg_sum_workspace(), dtype=torch.uint8, device=dev)
        self._ones = None

    @staticmethod
    def split(Wcat):
        """(Theta, Phi) views of a layer's [Theta | Phi]."""
        C = Wcat.shape[1] // 2
        return Wcat[:, :C], Wcat[:, C:]

    def train_step(self, H: torch.Tensor, lr: float = 0.0):
        from .ops import edgeconv_backward_cat, edgeconv_forward_cat

        xs, stashes = [H], []
        for Wcat in self.layers:
            out, st = edgeconv_forward_cat(self.g, xs[-1], Wcat)
            xs.append(out)
            stashes.append(st)
        out = xs[-1]
        call("gnncg_sum", out.numel(), _ptr(out), _ptr(self.loss), _ptr(self._sum_ws), self._sum_ws.numel(), _stream())
        if self._ones is None or self._ones.shape != out.shape:
            self._ones = torch.empty_like(out)
            call("gnncg_fill", self._ones.numel(), 1.0, _ptr(self._ones), _stream())
        g = self._ones
        grads = [None] * len(self.layers)
        for i in reversed(range(len(self.layers))):
            dH, dWcat = edgeconv_backward_cat(self.g, xs[i], self.layers[i], stashes[i], g, need_dH=i > 0)
            grads[i] = self.split(dWcat)
            g = dH
        for Wcat, (dTh, dPh) in zip(self.layers, grads):
            # dTh / dPh are the halves of one contiguous d[Theta | Phi]: one update
            call("gnncg_sgd_update", Wcat.numel(), lr, _ptr(dTh), _ptr(Wcat), _stream())
        return self.loss[:1], grads


class MoNet:
    """GMMConv stack: dims = [F0, F1, ...] with K kernels and r pseudo-coordinate
    dimensions per layer; identity between layers, loss = sum of exits, SGD on W, P_l, P_r, mu, sinv.
    W, P_l and P_r of a layer are column blocks of one row-padded parameter buffer
    [W | P_l | P_r | 0] (ops.gmm_weight_width), so neither the forward nor the backward copies."""

    def __init__(self, g: DeviceGraph, dims, K: int, r: int, seed: int = 0):
        from .ops import gmm_weight_width

        self.g, self.K, self.r = g, K, r
        dev = g.device
        gen = torch.Generator(device=dev)
        gen.manual_seed(seed)
        self.layers = []
        for a, b in zip(dims[:-1], dims[1:]):
            sinv = torch.rand(K, r, generator=gen, device=dev).add_(0.5)
            W, Pl, Pr = init_uniform(a, K * b, gen, dev), init_uniform(a, r, gen, dev), init_uniform(a, r, gen, dev)
            mu = init_uniform(K, r, gen, dev)
            Wcat = torch.zeros(a, gmm_weight_width(K, r, b), device=dev)  # once, at init
            Kf = K * b
            Wcat[:, :Kf], Wcat[:, Kf:Kf + r], Wcat[:, Kf + r:Kf + 2 * r] = W, Pl, Pr
            self.layers.append([Wcat, mu, sinv, b])
        self.loss = torch.zeros(4, device=dev)
        self._sum_ws = torch.empty(_lib.lib().gnncg_sum_workspace(), dtype=torch.uint8, device=dev)
        self._ones = None

    def views(self, Wcat, f):
        """(W, P_l, P_r) column views of a layer's [W | P_l | P_r | 0]."""
        Kf, r = self.K * f, self.r
        return Wcat[:, :Kf], Wcat[:, Kf:Kf + r], Wcat[:, Kf + r:Kf + 2 * r]

    def train_step(self, H: torch.Tensor, lr: float = 0.0):
        from .ops import gmm_backward, gmm_forward

        xs, stashes = [H], []
        for Wcat, mu, sinv, f in self.layers:
            out, st = gmm_forward(self.g, xs[-1], *self.views(Wcat, f), mu, sinv, self.K, self.r, f)
            xs.append(out)
            stashes.append(st)
        out = xs[-1]
        call("gnncg_sum", out.numel(), _ptr(out), _ptr(self.loss), _ptr(self._sum_ws), self._sum_ws.numel(), _stream())
        if self._ones is None or self._ones.shape != out.shape:
            self._ones = torch.empty_like(out)
            call("gnncg_fill", self._ones.numel(), 1.0, _ptr(self._ones), _stream())
        g = self._ones
        grads = [None] * len(self.layers)
        for i in reversed(range(len(self.layers))):
            Wcat, mu, sinv, f = self.layers[i]
            res = gmm_backward(self.g, xs[i], *self.views(Wcat, f), mu, sinv, self.K, self.r, f, stashes[i], g,
                               need_dH=i > 0)
            grads[i] = res[1:]
            g = res[0]
        for (Wcat, mu, sinv, f), gr in zip(self.layers, grads):
            dWcat, dmu, dsinv = gr[5], gr[3], gr[4]
            call("gnncg_sgd_update", Wcat.numel(), lr, _ptr(dWcat), _ptr(Wcat), _stream())
            call("gnncg_sgd_update", mu.numel(), lr, _ptr(dmu), _ptr(mu), _stream())
            call("gnncg_sgd_update", sinv.numel(), lr, _ptr(dsinv), _ptr(sinv), _stream())
        return self.loss[:1], grads


class GCN:
    """Vanilla GCN stack: h' = relu(b + sum_e w_e h_u W) per
    layer with the symmetric edge normalisation, loss = sum of exits, SGD on W and b."""

    def __init__(self, g: DeviceGraph, dims, seed: int = 0, chunk: int | None = None):
        from .ops import gcn_norm

        self.g, self.chunk = g, chunk
        dev = g.device
        gen = torch.Generator(device=dev)
        gen.manual_seed(seed)
        self.layers = [(init_uniform(a, b, gen, dev), init_uniform(1, b, gen, dev).view(b))
                       for a, b in zip(dims[:-1], dims[1:])]
        self.edge_w = gcn_norm(g)
        self.loss = torch.zeros(4, device=dev)
        self._sum_ws = torch.empty(_lib.lib().gnncg_sum_workspace(), dtype=torch.uint8, device=dev)

    def train_step(self, H: torch.Tensor, lr: float = 0.0):
        from .ops import gcn_backward, gcn_forward

        xs, stashes = [H], []
        for W, b in self.layers:
            out, st = gcn_forward(self.g, xs[-1], W, b, self.edge_w, chunk=self.chunk)
            xs.append(out)
            stashes.append(st)
        out = xs[-1]
        call("gnncg_sum", out.numel(), _ptr(out), _ptr(self.loss), _ptr(self._sum_ws), self._sum_ws.numel(), _stream())
        g = torch.empty_like(out)
        call("gnncg_fill", g.numel(), 1.0, _ptr(g), _stream())
        grads = [None] * len(self.layers)
        for i in reversed(range(len(self.layers))):
            W, b = self.layers[i]
            dH, dW, db = gcn_backward(self.g, xs[i], W, stashes[i], g, self.edge_w, need_dH=i > 0, chunk=self.chunk)
            grads[i] = (dW, db)
            g = dH
        for (W, b), (dW, db) in zip(self.layers, grads):
            call("gnncg_sgd_update", W.numel(), lr, _ptr(dW), _ptr(W), _stream())
            call("gnncg_sgd_update", b.numel(), lr, _ptr(db), _ptr(b), _stream())
        return self.loss[:1], grads


class GraphedStep:
    """A training step captured once into a CUDA graph and replayed (launch-bound small graphs).

    The model's train_step(H, lr) is recorded on a side stream with the input in a static buffer;
    replay() re-runs every kernel of the step (forward, loss, backward, SGD) with one launch.
    Device allocations made inside the step come from the graph's private memory pool."""

    def __init__(self, model, H_static: torch.Tensor, lr: float, warmup: int = 2):
        self.model, self.H, self.lr = model, H_static, lr
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(warmup):
                model.train_step(H_static, lr=lr)
        torch.cuda.current_stream().wait_stream(s)
        self.graph = torch.cuda.CUDAGraph()
        n0 = _lib.lib().gnncg_launch_count()
        with torch.cuda.graph(self.graph):
            self.loss, self.grads = model.train_step(H_static, lr=lr)
        self.kernels = int(_lib.lib().gnncg_launch_count() - n0)  # library kernels per replay

    def replay(self):
        self.graph.replay()
        return self.loss, self.grads
