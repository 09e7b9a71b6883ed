"""GPU: measured == predicted (acceptance criterion 9).  The device cost
counters (gnncg_cost_counters) record, per kernel kind, the edges every work item walked and
the rows completed; flops and io units follow from the kernels' fixed per-edge / per-row work
(cost.py) and must equal the closed forms exactly, including on graphs whose hub rows are split
and whose items are fetched from the work counter.  Also the `compare` report."""
import json
import os

import numpy as np
import pytest
import torch

from paper_2110_09524_b200 import cost
from paper_2110_09524_b200.graph import DeviceGraph
from paper_2110_09524_b200.ops import GatParams
from paper_2110_09524_b200.report import gat_layer_report

pytestmark = pytest.mark.gpu


def _layer(cuda, g, fin, h, f, seed=0):
    gen = torch.Generator(device=cuda)
    gen.manual_seed(seed)
    V = g.num_vertices
    ld = (fin + 3) // 4 * 4
    H = (torch.rand(V, ld, generator=gen, device=cuda) * 2 - 1)[:, :fin]
    W = (torch.rand(fin, h * f, generator=gen, device=cuda) - 0.5) / np.sqrt(fin)
    a_l = torch.rand(h, f, generator=gen, device=cuda) - 0.5
    a_r = torch.rand(h, f, generator=gen, device=cuda) - 0.5
    return H, W, a_l, a_r


CASES = [
    ("G3", lambda dev: DeviceGraph.from_edges(3, np.array([0, 1, 0]), np.array([2, 2, 1]), device=dev), 4, 1, 2),
    ("erdos_renyi_100", lambda dev: DeviceGraph.from_edges(100, *_er(100, 0.05, 1), device=dev), 12, 2, 4),
    ("chung_lu_hubs_f32", lambda dev: DeviceGraph.chung_lu(20_000, 2_000_000, offset=30, seed=1, device=dev), 64, 8, 32),
    ("chung_lu_hubs_f16", lambda dev: DeviceGraph.chung_lu(20_000, 2_000_000, offset=30, seed=2, device=dev), 64, 8, 16),
]


def _er(V, p, seed):
    rng = np.random.default_rng(seed)
    a = rng.random((V, V)) < p
    np.fill_diagonal(a, False)
    s, d = np.nonzero(a)
    return s, d


@pytest.mark.parametrize("name,make,fin,h,f", CASES, ids=[c[0] for c in CASES])
def test_counters_equal_closed_forms(cuda, name, make, fin, h, f):
    g = make(cuda)
    V, E = g.num_vertices, g.num_edges
    rep = gat_layer_report(g, *_layer(cuda, g, fin, h, f), GatParams(h, f), config={"graph": name, "h": h, "f": f})
    c = rep["counters"]
    assert c["edges"]["K2"] == E and c["rows"]["K2"] == V and c["lp_rows"] == V, c
    if c["edges"]["K4f"]:
        assert c["edges"]["K4f"] == E and c["rows"]["K4f"] == V, c
    allr = rep["results"][-1]
    assert allr["opt"] == "all" and all(v for k, v in allr["checks"].items()), allr
    assert allr["flops"] == cost.gat_executed_flops(V, E, h, f)
    if name == "G3":  # 39 -> 30 flops, 45 -> 33 io units (paper formulas)
        assert [r["flops"] for r in rep["results"][:2]] == [39, 30]
        assert rep["results"][0]["io_units"] == 45 and rep["results"][2]["io_units"] == 33
        assert allr["flops"] == 30
    if name == "chung_lu_hubs_f32":
        os.makedirs("gpurun_out", exist_ok=True)
        with open("gpurun_out/compare_report.json", "w") as fh:
            json.dump(rep, fh, indent=1)
