"""GPU: the tcgen05/TMA 3xTF32 GEMM (K1/K5) against float64 -- every operand major
(NN, NT, TN), M/N/K tails, split-K, and agreement with the CUDA-core path."""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from paper_2110_09524_b200 import gemm

pytestmark = pytest.mark.gpu


def padded(rows, cols, dev, rng):
    ld = (cols + 3) // 4 * 4
    buf = torch.empty(rows, ld, device=dev, dtype=torch.float32)
    buf[:, :cols] = torch.from_numpy(rng.uniform(-1, 1, (rows, cols)).astype(np.float32)).to(dev)
    return buf[:, :cols]


CASES = [  # (trans_a, trans_b, M, N, K)
    (0, 0, 4096, 256, 604), (0, 0, 233, 256, 256), (0, 0, 1000, 128, 100), (0, 0, 300, 64, 32),
    (0, 1, 2048, 256, 256), (0, 1, 777, 96, 64), (0, 1, 5000, 604, 256),
    (1, 0, 604, 256, 20000), (1, 0, 256, 256, 50000), (1, 0, 130, 128, 3000), (0, 0, 129, 17, 5),
    # tall products with a small reused B: B's tf32 lo part is pre-split once into the workspace
    (0, 0, 20000, 256, 602), (0, 1, 20003, 604, 256), (0, 0, 16500, 128, 100),
]


@pytest.mark.parametrize("ta,tb,M,N,K", CASES)
def test_tc_gemm_vs_f64(cuda, ta, tb, M, N, K):
    rng = np.random.default_rng(M * 7 + N * 3 + K)
    A = padded(K, M, cuda, rng) if ta else padded(M, K, cuda, rng)
    B = padded(N, K, cuda, rng) if tb else padded(K, N, cuda, rng)
    C = gemm(A, B, trans_a=bool(ta), trans_b=bool(tb))
    torch.cuda.synchronize()
    a = A.double().T if ta else A.double()
    b = B.double().T if tb else B.double()
    ref = (a @ b).cpu().numpy()
    err = np.abs(C.double().cpu().numpy() - ref).max() / max(1.0, np.abs(ref).max())
    # 3xTF32 keeps ~21 mantissa bits per product; what remains is fp32 accumulation over K
    # (measured 3e-6 at K=256 .. 2.3e-5 at K=50000, max-normalised): inside the 1e-4 path bound
    assert err < 5e-5, err


def test_tc_and_simt_agree(cuda):
    """Run the same product under GNNCG_GEMM=simt in a subprocess and compare."""
    code = (
        "import torch,numpy as np,sys;sys.path.insert(0,'.');from paper_2110_09524_b200 import gemm;"
        "g=torch.Generator(device='cuda');g.manual_seed(0);"
        "b=torch.rand(3000,604,device='cuda',generator=g);A=b[:,:602];W=torch.rand(602,256,device='cuda',generator=g);"
        "C=gemm(A,W);torch.cuda.synchronize();np.save(sys.argv[1],C.cpu().numpy())")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for mode in ("tc", "simt"):
        path = f"/tmp/gemm_{mode}.npy"
        env = dict(os.environ, GNNCG_GEMM=mode)
        subprocess.run([sys.executable, "-c", code, path], cwd=root, env=env, check=True, timeout=300)
        outs.append(np.load(path))
    assert np.abs(outs[0] - outs[1]).max() < 2e-5 * max(1.0, np.abs(outs[1]).max())


@pytest.mark.parametrize("tc", ["tc", "simt"])
def test_gemm_tall_m_beyond_grid_y(cuda, tc, monkeypatch):
    """M > 65535 * 128 rows (C5: 10M vertices): M tiles are on gridDim.x."""
    M, N, K = 9_000_000, 16, 16
    if tc == "simt":
        A = torch.ones(M, K + 1, device=cuda)[:, :K]  # unaligned ld -> CUDA-core path
    else:
        A = torch.ones(M, K, device=cuda)
    B = torch.full((K, N), 0.5, device=cuda)
    C = gemm(A, B)
    torch.cuda.synchronize()
    assert C.min().item() == 8.0 and C.max().item() == 8.0


@pytest.mark.parametrize("M,K,h,f", [(1000, 602, 8, 32), (4097, 256, 8, 32), (777, 64, 4, 64), (300, 100, 2, 32),
                                     (20000, 602, 8, 32),
                                     (513, 128, 8, 16), (50, 20, 3, 5)])
def test_gat_transform_epilogue(cuda, M, K, h, f):
    """K1 with the attention-LP epilogue equals gemm + attn_dots bitwise (fused when f % 32 == 0,
    the unfused pair otherwise)."""
    from paper_2110_09524_b200.ops import attn_dots, gat_transform, gemm
    g = torch.Generator(device=cuda)
    g.manual_seed(M + K)
    ld = (K + 3) // 4 * 4
    Hb = torch.rand(M, ld, generator=g, device=cuda) * 2 - 1
    H = Hb[:, :K]
    W = (torch.rand(K, h * f, generator=g, device=cuda) * 2 - 1) / K ** 0.5
    al = torch.rand(h, f, generator=g, device=cuda) - 0.5
    ar = torch.rand(h, f, generator=g, device=cuda) - 0.5
    Ht, Al, Ar = gat_transform(H, W, al, ar, h, f)
    Ht2 = gemm(H, W)
    Al2, Ar2 = attn_dots(Ht2, al, ar, h, f)
    torch.cuda.synchronize()
    assert torch.equal(Ht, Ht2)
    assert torch.equal(Al, Al2)
    assert torch.equal(Ar, Ar2)


@pytest.mark.parametrize("ta,tb", [(0, 0), (0, 1), (1, 0)])
def test_tc_gemm_identity_split(cuda, ta, tb):
    """C = A I reproduces every element of A to 2^-20 relative.  This pins the 3xTF32 split the
    kernel relies on (a = hi + lo, hi = a with the low 13 mantissa bits cleared): the only loss
    left is lo's own conversion to tf32 (<= 2^-21 |a|).  A split whose hi were ROUNDED rather
    than truncated by the tensor core would leave up to 2^-11 |a| on about half of the entries."""
    rng = np.random.default_rng(11)
    M, K = 640, 96
    A = padded(K, M, cuda, rng) if ta else padded(M, K, cuda, rng)
    I = torch.eye(K, device=cuda, dtype=torch.float32)
    C = gemm(A, I, trans_a=bool(ta), trans_b=bool(tb))
    torch.cuda.synchronize()
    ref = (A.T if ta else A).double()
    rel = ((C.double() - ref).abs() / ref.abs().clamp_min(1e-30)).max().item()
    assert rel <= 2.0 ** -20, rel
