"""paper_2110_09524_b200 -- B200-native (sm_100a) fused GNN layer path of arXiv 2110.09524.

Drop-in for the reference's fused GAT / EdgeConv / GMMConv (+ GCN) layer path
(SPEC.md:316-390 executor; proj/include/gnncg graph and tensor model).  All
compute runs in the in-tree ``libgnncg_b200.so`` (C ABI: include/gnncg_b200.h);
there is no CPU fallback.
"""
from ._lib import (ArgumentError, CudaError, DeviceError, GnncgError, GraphError, TensorError,  # noqa: F401
                   UnsupportedError, WorkspaceError, hot_window, l2_persist)
from .graph import (DeviceGraph, DeviceIndex, DeviceSched, chung_lu_cdf, knn_edges, partition_rows,  # noqa: F401
                    permute_rows, uniform_edges, unpermute_rows)
from .ops import (GatGrads, GatParams, GatStash, edgeconv_backward, edgeconv_forward, gat_backward,  # noqa: F401
                  gat_forward, gat_region_backward, gat_region_forward, gcn_backward, gcn_forward, gcn_norm, gemm,
                  gmm_backward, gmm_forward, matmul, matmul_nt, matmul_tn, spmm)

__version__ = "0.1.0"
