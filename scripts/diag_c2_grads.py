"""Diagnose the C2 gradient parity: GPU fast / deterministic backward, the f32 CPU port and the
f64 oracle on the Reddit-shaped graph; per tensor: max |ref|, max abs err, elementwise rel_err,
and the rel_err of the f32 port (the conditioning of the fp32 computation itself)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import oracle as O  # noqa: E402
from paper_2110_09524_b200.graph import DeviceGraph  # noqa: E402
from paper_2110_09524_b200.models import GAT  # noqa: E402
from tests.test_gpu_scale import features, host_graph, np64  # noqa: E402

scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
dev = torch.device("cuda:0")
V, E = int(233000 * scale), int(114000000 * scale)
g = DeviceGraph.chung_lu(V, E, offset=max(1, int(1100 * scale)), seed=0, device=dev)
dims = [(602, 8, 32), (256, 8, 32)]
res = {}
for mode in ("fast", "deterministic"):
    model = GAT(g, dims, seed=1, mode=mode)
    H = features(V, 602, dev)
    xs, st = model.forward(H)
    gr = model.backward(xs, st, model.seed_grad(xs[-1]))
    torch.cuda.synchronize()
    res[mode] = {"dW1": np64(gr[0].dW), "dal1": np64(gr[0].da_l), "dar1": np64(gr[0].da_r), "dW2": np64(gr[1].dW),
                 "dal2": np64(gr[1].da_l), "dar2": np64(gr[1].da_r), "dH2": np64(gr[1].dH)}
hg = host_graph(g)
Hh = np64(H)
out = {}
for dt in (np.float64, np.float32):
    t0 = time.time()
    fws, ins = [], [Hh]
    for L in model.layers:
        fw = O.gat_layer_fwd_omp(hg, ins[-1], np64(L.W), np64(L.a_l), np64(L.a_r), 8, 32, dtype=dt)
        fws.append(fw)
        ins.append(fw["out"])
    b2 = O.gat_layer_bwd_omp(hg, ins[1], np64(model.layers[1].W), np64(model.layers[1].a_l), np64(model.layers[1].a_r),
                             8, 32, fws[1], np.ones_like(ins[2]), True, dtype=dt)
    b1 = O.gat_layer_bwd_omp(hg, ins[0], np64(model.layers[0].W), np64(model.layers[0].a_l), np64(model.layers[0].a_r),
                             8, 32, fws[0], b2["dH"], False, dtype=dt)
    out[dt] = {"dW1": b1["dW"], "dal1": b1["dal"], "dar1": b1["dar"], "dW2": b2["dW"], "dal2": b2["dal"],
               "dar2": b2["dar"], "dH2": b2["dH"], "dAl1": b1["dAl"], "dAr1": b1["dAr"], "c1": b1["c"]}
    print(dt.__name__, "oracle s", time.time() - t0, flush=True)
ref = out[np.float64]
for k in ("dW2", "dal2", "dar2", "dH2", "dW1", "dal1", "dar1"):
    r = ref[k].astype(np.float64)
    line = [k, f"max|ref| {np.abs(r).max():.3e}"]
    for name, got in (("fast", res["fast"][k]), ("det", res["deterministic"][k]), ("cpu_f32", out[np.float32][k])):
        a = np.abs(got - r)
        line.append(f"{name}: abs {a.max():.2e} rel {O.max_rel_err(got, r):.2e} maxnorm {a.max() / max(1, np.abs(r).max()):.2e}")
    print(" | ".join(line), flush=True)
for k in ("dAl1", "dAr1", "c1"):
    print(k, "max|.|", np.abs(ref[k]).max(), "f32 abs err", np.abs(out[np.float32][k] - ref[k]).max())
print("max |dH2| (layer-1 dOut)", np.abs(ref["dH2"]).max())
