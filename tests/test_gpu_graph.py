"""GPU: device graph store (K9) is bit-exact with the reference's build_index."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2110_09524_b200 import DeviceGraph, GraphError
from paper_2110_09524_b200.graph import chung_lu_edges_host
from tests.conftest import golden_graphs

pytestmark = pytest.mark.gpu

FIELDS = ("dst_off", "dst_src", "dst_eid", "src_off", "src_dst", "src_eid")


def test_csr_build_matches_reference_goldens(cuda, golden):
    for name, d in golden_graphs(golden):
        g = DeviceGraph.from_edges(d["V"], d["src"], d["dst"], device=cuda)
        h = g.to_host()
        for f in FIELDS:
            np.testing.assert_array_equal(h[f], d[f], err_msg=f"{name}:{f}")
        mi, mean, mo = g.degree_stats()
        assert (mi, mean, mo) == (d["stats"][0], d["stats"][1], d["stats"][2]), name


@pytest.mark.parametrize("V,E", [(1, 1000), (64, 0), (1000, 100000), (100000, 3000000)])
def test_csr_build_random_bit_exact(cuda, V, E):
    rng = np.random.default_rng(V + E)
    src, dst = rng.integers(0, V, E), rng.integers(0, V, E)
    g = DeviceGraph.from_edges(V, src, dst, device=cuda)
    ref = O.host_graph(V, src, dst)
    h = g.to_host()
    for f in FIELDS:
        np.testing.assert_array_equal(h[f], getattr(ref, f), err_msg=f)


def test_csr_build_rejects_out_of_range(cuda):
    with pytest.raises(GraphError):
        DeviceGraph.from_edges(4, [0, 1, 4], [1, 2, 3], device=cuda)  # graph.cpp:37-39


def test_chung_lu_device_matches_host_restatement(cuda):
    V, E, off, seed = 5000, 20000, 50, 3
    g = DeviceGraph.chung_lu(V, E, offset=off, seed=seed, device=cuda)
    src, dst = chung_lu_edges_host(V, E, off, seed)
    np.testing.assert_array_equal(g.edge_src.cpu().numpy().view(np.uint32), src)
    np.testing.assert_array_equal(g.edge_dst.cpu().numpy().view(np.uint32), dst)
    ref = O.host_graph(V, src, dst)
    h = g.to_host()
    for f in FIELDS:
        np.testing.assert_array_equal(h[f], getattr(ref, f))


def test_chung_lu_is_skewed(cuda):
    g = DeviceGraph.chung_lu(20000, 2_000_000, offset=100, seed=0, device=cuda)
    mi, mean, mo = g.degree_stats()
    assert mean == 100.0 and mi > 10 * mean and mo > 10 * mean
    torch.cuda.synchronize()
