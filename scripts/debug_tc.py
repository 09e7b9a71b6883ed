"""Focused tcgen05 GEMM probe: tiny shapes, constant and random operands, every major."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2110_09524_b200 import gemm

dev = torch.device("cuda")
print("dbg", os.environ.get("GNNCG_TC_DEBUG"))
for ta, tb, M, N, K in [(0, 1, 128, 256, 32), (0, 1, 128, 128, 32), (0, 0, 128, 256, 64), (1, 0, 128, 256, 64)]:
    A = torch.ones(K, M, device=dev) if ta else torch.ones(M, K, device=dev)
    B = torch.ones(N, K, device=dev) if tb else torch.ones(K, N, device=dev)
    C = gemm(A, B, trans_a=bool(ta), trans_b=bool(tb))
    torch.cuda.synchronize()
    c = C.cpu().numpy()
    print(ta, tb, M, N, K, "ones ->", c[0, :4], c[M - 1, N - 4:], "nonzero frac", (c != 0).mean())
    g = torch.Generator(device=dev); g.manual_seed(0)
    A = torch.rand(A.shape, device=dev, generator=g) - 0.5
    B = torch.rand(B.shape, device=dev, generator=g) - 0.5
    C = gemm(A, B, trans_a=bool(ta), trans_b=bool(tb))
    ref = (A.double().T if ta else A.double()) @ (B.double().T if tb else B.double())
    torch.cuda.synchronize()
    print("   rand err", (C.double() - ref).abs().max().item(), "ref max", ref.abs().max().item())
