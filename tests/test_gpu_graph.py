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


@pytest.mark.parametrize("P", [1, 3, 8])
def test_per_rank_chung_lu_equals_filtered_global_list(cuda, P):
    """Multi-GPU graph build: each rank's edges (gnncg_gen_chung_lu_rows) are the global edge
    list filtered to its destination block, in edge-id order; the in-degree histogram and the
    row bounds equal those of the global list; the local CSR is the global CSR's row block."""
    from paper_2110_09524_b200.dist import DEFAULT_ROW_WEIGHT, partitioned_chung_lu

    V, E, off, seed = 20000, 1_000_000, 100, 5
    src, dst = chung_lu_edges_host(V, E, off, seed)
    ref = O.host_graph(V, src, dst)
    # the multi-GPU default: cost-balanced blocks (gnncg_partition_rows_weighted)
    bounds = O.partition_rows_weighted(ref.dst_off, P, DEFAULT_ROW_WEIGHT)
    total = 0
    for rank in range(P):
        lg = partitioned_chung_lu(V, E, offset=off, seed=seed, rank=rank, world=P, device=cuda)
        np.testing.assert_array_equal(lg.plan.bounds, bounds)
        r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
        mr, base, n = lg.plan.maxrows, lg.row_base, r1 - r0
        ref_off = ref.dst_off[r0:r1 + 1].astype(np.int64)
        ref_src = ref.dst_src[ref.dst_off[r0]:ref.dst_off[r1]].astype(np.int64)
        ref_row = np.repeat(np.arange(n), np.diff(ref_off))
        own = (ref_src >= r0) & (ref_src < r1)
        # local source ids live in the padded all-gather layout: map back to global ids
        pid_to_global = lambda pid: lg.plan.bounds[pid // mr].astype(np.int64) + pid % mr  # noqa: E731
        for idx, sel in ((lg.csr_local, own), (lg.csr_remote, ~own)):
            loff, lnbr, _ = idx.to_host()
            # each part is the global row block filtered by source owner, in edge-id order
            np.testing.assert_array_equal(np.diff(loff.astype(np.int64)), np.bincount(ref_row[sel], minlength=n))
            np.testing.assert_array_equal(pid_to_global(lnbr.astype(np.int64)), ref_src[sel])
        # csc_local: own sources rebased to the block, rows sorted by source then edge id
        coff, cnbr, _ = lg.csc_local.to_host()
        np.testing.assert_array_equal(np.diff(coff.astype(np.int64)), np.bincount(ref_src[own] - r0, minlength=n))
        assert lg.csc_remote.num_rows == lg.plan.padded_V and lg.csc_remote.num_edges == int((~own).sum())
        total += int(lg.num_edges)
    assert total == E
