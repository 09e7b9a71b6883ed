"""Diagnostic (GPU): where does the C2 bench step's loss become non-finite under SGD?
Runs the bench's model step by step and reports loss, parameter / output / gradient
magnitudes and the first non-finite tensor.  usage: python scripts/diag_nan.py [lr] [steps] [mode]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2110_09524_b200.graph import DeviceGraph  # noqa: E402
from paper_2110_09524_b200.models import GAT  # noqa: E402

lr = float(sys.argv[1]) if len(sys.argv) > 1 else 1e-6
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 15
mode = sys.argv[3] if len(sys.argv) > 3 else "auto"
dev = torch.device("cuda:0")
g = DeviceGraph.chung_lu(233_000, 114_000_000, offset=1100, seed=0, device=dev)
model = GAT(g, [(602, 8, 32), (256, 8, 32)], seed=1, mode=mode)
gen = torch.Generator(device=dev)
gen.manual_seed(1234)
H = torch.rand(233_000, 604, generator=gen, device=dev).mul_(2).sub_(1)[:, :602]


def mx(t):
    return float(t.abs().max()) if torch.isfinite(t).all() else float("nan")


for i in range(steps):
    xs, st = model.forward(H)
    out = xs[-1]
    loss = float(out.double().sum())
    grads = model.backward(xs, st, model.seed_grad(out))
    info = {"loss": loss, "out1": mx(xs[1]), "out2": mx(xs[2])}
    for j, (L, gr) in enumerate(zip(model.layers, grads)):
        info[f"W{j + 1}"] = mx(L.W)
        info[f"al{j + 1}"] = mx(L.a_l)
        info[f"dW{j + 1}"] = mx(gr.dW)
        info[f"dal{j + 1}"] = mx(gr.da_l)
        info[f"dar{j + 1}"] = mx(gr.da_r)
        if gr.dH is not None:
            info[f"dH{j + 1}"] = mx(gr.dH)
        for k, s in (("m", st[j].m), ("d", st[j].d)):
            info[f"{k}{j + 1}"] = mx(s)
    print(i, {k: f"{v:.3e}" for k, v in info.items()}, flush=True)
    if any(v != v for v in info.values()):
        break
    model.sgd(grads, lr)
torch.cuda.synchronize()
