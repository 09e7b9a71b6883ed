"""Per-rank compute of the row-partitioned GAT step, one rank at a time on ONE GPU.

Each rank r of a P-way partition builds only its own share of the graph (partitioned_chung_lu)
and runs the PartitionedGAT training step through the library's dist entry points
(gnncg_gat_fwd_dist / gnncg_gat_bwd_dist) with no communicator: the all-gather, the
reduce-scatter and the parameter all-reduce are skipped (the remote gather-table rows are left
unfilled, so the numbers are timings only).  What it shows: how evenly the partitioner splits
the work (max vs mean per-rank step) and the compute floor of a P-GPU step; the collectives'
volume is printed beside it.  It is NOT a multi-GPU measurement.

usage: python scripts/emulate_ranks.py --config c5 --parts 8 [--steps 3 --warmup 2]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2110_09524_b200 import _lib  # noqa: E402
from paper_2110_09524_b200.dist import PartitionedGAT, partitioned_chung_lu  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", choices=["c5", "reddit"], default="c5")
    ap.add_argument("--parts", type=int, default=8)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--l2-persist-mb", type=int, default=48)
    ap.add_argument("--row-weight", type=int, default=None, help="partitioner row weight (default: dist's)")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    _lib.l2_persist(args.l2_persist_mb << 20)
    if args.config == "c5":
        V, E, offset, dims = 10_000_000, 1_000_000_000, 10_000, [(128, 8, 16)] * 3
    else:
        V, E, offset, dims = 233_000, 114_000_000, 1100, [(602, 8, 32), (256, 8, 32)]
    per = []
    for r in range(args.parts):
        kw = {} if args.row_weight is None else {"row_weight": args.row_weight}
        lg = partitioned_chung_lu(V, E, offset=offset, seed=0, rank=r, world=args.parts, device=dev, **kw)
        model = PartitionedGAT(lg, dims, seed=1)
        gen = torch.Generator(device=dev).manual_seed(1234 + r)
        fin = dims[0][0]
        ld = (fin + 3) // 4 * 4  # 16-byte aligned rows for the TMA GEMM (as bench.py)
        H = (torch.rand(lg.num_local, ld, generator=gen, device=dev) * 2 - 1)[:, :fin]
        for _ in range(args.warmup):
            model.train_step(H, lr=1e-10)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(args.steps):
            model.train_step(H, lr=1e-10)
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / args.steps
        per.append({"rank": r, "rows": lg.num_local, "edges": lg.num_edges, "ms_per_step": ms})
        print(json.dumps(per[-1]), flush=True)
        del model, lg, H
        torch.cuda.empty_cache()
    hf_h = sum(h * f + h for _, h, f in dims)
    mx = max(p["ms_per_step"] for p in per)
    mean = sum(p["ms_per_step"] for p in per) / len(per)
    out = {"config": args.config, "parts": args.parts, "row_weight": args.row_weight, "V": V, "E": E,
           "maxrows": max(p["rows"] for p in per), "max_rank_ms": mx, "mean_rank_ms": mean,
           "balance": mean / mx, "edges_per_s_compute_floor": E * len(dims) / (mx / 1e3),
           "allgather_bytes_per_rank_per_step": int(V * hf_h * 4 * (args.parts - 1) / args.parts),
           "note": "per-rank compute only, collectives skipped (no communicator); not a multi-GPU measurement",
           "ranks": per}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
