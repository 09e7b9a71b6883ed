"""GPU: the compiled plan drives the real kernels -- compile_model(...).model(g) runs a training
step identical (bitwise) to the hand-built model on the same kernels."""
import pytest
import torch

from paper_2110_09524_b200 import DeviceGraph
from paper_2110_09524_b200 import ir as I
from paper_2110_09524_b200.models import GAT

pytestmark = pytest.mark.gpu


def test_compiled_gat_drives_the_kernels(cuda):
    V, E, dims = 2000, 40000, [(48, 8, 32)]
    g = DeviceGraph.chung_lu(V, E, offset=30, seed=2, device=cuda)
    c = I.compile_model("gat", max_in_degree=1000, mean_in_degree=E / V)
    assert c.plan.names()[0].startswith("gnncg_gat_transform")
    gen = torch.Generator(device=cuda)
    gen.manual_seed(1)
    H = torch.rand(V, 48, generator=gen, device=cuda)
    a = c.model(g, dims, seed=3, mode="deterministic")
    b = GAT(g, dims, seed=3, mode="deterministic")
    la, ga = a.train_step(H)
    lb, gb = b.train_step(H)
    torch.cuda.synchronize()
    assert torch.equal(la, lb)
    for x, y in zip(ga, gb):
        assert torch.equal(x.dW, y.dW) and torch.equal(x.da_l, y.da_l) and torch.equal(x.da_r, y.da_r)
