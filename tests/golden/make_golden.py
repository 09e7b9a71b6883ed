"""Generate tests/golden/reference_golden.npz from the reference's OWN code.

Runs only where /root/reference exists (this container): oracle/Makefile compiles
/root/reference/proj/src/{graph,tensor}.cpp into oracle/_ref/libgnncg_ref.so and
this script records what that code produces, so the GPU box (which has no
/root/reference) can check against committed vectors:

  * Graph(V, edges) -> csr_dst / csc_src (graph.cpp:14-45) for the spec's fixture
    graphs (G3), descriptor graphs via generate_synthetic
    (graph.cpp:157-249: star, k_regular_in, erdos_renyi with the seeds the spec's
    test matrix uses), and a few random edge lists with
    duplicates / isolated vertices;
  * degree_stats (graph.cpp:47-57);
  * init_seeded<T> (tensor.hpp:44-63);
  * matmul / matmul_nt / matmul_tn (tensor.cpp:8-60) on small random operands.

Usage:  python tests/golden/make_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_golden.npz")

DESCRIPTORS = [("star:4", 0), ("star:5:2", 0), ("star:1000", 0), ("k_regular_in:5:2", 42), ("k_regular_in:32:4", 42),
               ("erdos_renyi:10:0.3", 1), ("erdos_renyi:16:0.3", 7), ("erdos_renyi:100:0.05", 1)]


def main():
    if not O.ref_available():
        raise SystemExit("oracle/_ref/libgnncg_ref.so missing: run `make -C oracle` with /root/reference present")
    data = {}
    cases = []

    def add(name, g: O.RefGraph):
        hg = g.to_host()
        mi, mean, mo = g.degree_stats()
        key = f"g{len(cases)}"
        cases.append(name)
        data[f"{key}_V"] = np.array([hg.V], np.uint64)
        for fld in ("src", "dst", "dst_off", "dst_src", "dst_eid", "src_off", "src_dst", "src_eid"):
            data[f"{key}_{fld}"] = getattr(hg, fld)
        data[f"{key}_stats"] = np.array([mi, mean, mo], np.float64)

    add("G3", O.RefGraph.from_edges(3, [0, 1, 0], [2, 2, 1]))
    add("empty", O.RefGraph.from_edges(0, [], []))
    add("isolated", O.RefGraph.from_edges(7, [0, 0, 6], [1, 1, 0]))  # duplicates kept, isolated vertices
    for desc, seed in DESCRIPTORS:
        add(f"{desc}@{seed}", O.RefGraph.synthetic(desc, seed))
    rng = np.random.default_rng(2110)
    for V, E in ((50, 400), (300, 5000), (1000, 20000)):
        src = rng.integers(0, V, E)
        dst = rng.integers(0, V, E)
        add(f"random:{V}:{E}", O.RefGraph.from_edges(V, src, dst))
    data["cases"] = np.array(cases)

    data["init_f64_2x3_42"] = O.ref_init_seeded(2, 3, 42, np.float64)
    data["init_f32_4x4_42"] = O.ref_init_seeded(4, 4, 42, np.float32)
    data["init_f64_16x8_7"] = O.ref_init_seeded(16, 8, 7, np.float64)
    data["init_f64_ones"] = O.ref_init_seeded(1, 1, 0, np.float64, dist=2)

    A = rng.standard_normal((37, 29)).astype(np.float32)
    B = rng.standard_normal((29, 23)).astype(np.float32)
    Bt = rng.standard_normal((23, 29)).astype(np.float32)
    At = rng.standard_normal((29, 37)).astype(np.float32)
    data["mm_A"], data["mm_B"], data["mm_Bt"], data["mm_At"] = A, B, Bt, At
    data["mm_nn"] = O.ref_matmul("nn", A, B)
    data["mm_nt"] = O.ref_matmul("nt", A, Bt)
    data["mm_tn"] = O.ref_matmul("tn", At, B)
    np.savez_compressed(OUT, **data)
    print(f"wrote {OUT}: {len(cases)} graphs")


if __name__ == "__main__":
    main()
