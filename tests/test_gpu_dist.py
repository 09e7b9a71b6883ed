"""GPU: the partitioned (multi-GPU) GAT through its real engine and NCCL collectives at
world size 1 (one GPU per box here) matches the single-GPU model step for step.  The
world-size 2/3 orchestration is covered on CPU by tests/test_dist_gloo.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture(scope="module", autouse=True)
def _nccl_teardown():
    yield
    if dist.is_initialized():
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["deterministic", "auto"])
def test_partitioned_world1_matches_single_gpu(cuda, mode):
    from paper_2110_09524_b200.dist import CudaEngine, PartitionedGAT, partitioned_chung_lu
    from paper_2110_09524_b200.graph import DeviceGraph
    from paper_2110_09524_b200.models import GAT

    if not dist.is_initialized():
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_port()}", rank=0, world_size=1,
                                device_id=cuda)
    V, E, dims = 3000, 120_000, [(64, 8, 16), (128, 8, 16)]
    lg = partitioned_chung_lu(V, E, offset=40, seed=5, rank=0, world=1, device=cuda)
    pm = PartitionedGAT(lg, dims, seed=7, engine=CudaEngine(cuda, mode=mode))
    g = DeviceGraph.chung_lu(V, E, offset=40, seed=5, device=cuda)
    sm = GAT(g, dims, seed=7, mode=mode)
    gen = torch.Generator(device=cuda)
    gen.manual_seed(3)
    H = torch.rand(V, 64, generator=gen, device=cuda) * 2 - 1
    lp, gp = pm.train_step(H, lr=0.0)
    ls, gs = sm.train_step(H, lr=0.0)
    torch.cuda.synchronize()
    assert abs(lp.item() - ls.item()) <= 1e-4 * max(1.0, abs(ls.item()))
    for (dW, da_l, da_r, _), gr in zip(gp, gs):
        for a, b in ((dW, gr.dW), (da_l, gr.da_l), (da_r, gr.da_r)):
            a, b = a.double().cpu().numpy(), b.double().cpu().numpy()
            s = max(1.0, np.abs(b).max())
            assert O.max_rel_err(a / s, b / s) < 1e-4
