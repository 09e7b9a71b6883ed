import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "reference_golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) -- run with -m gpu on the GPU box")


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLDEN)


def golden_graphs(z):
    """[(name, dict of arrays)] from the committed reference goldens."""
    out = []
    for i, name in enumerate(z["cases"]):
        k = f"g{i}"
        d = {f: z[f"{k}_{f}"] for f in ("src", "dst", "dst_off", "dst_src", "dst_eid", "src_off", "src_dst", "src_eid")}
        d["V"] = int(z[f"{k}_V"][0])
        d["stats"] = z[f"{k}_stats"]
        out.append((str(name), d))
    return out


@pytest.fixture(scope="session")
def cuda():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a B200"
    from paper_2110_09524_b200 import _lib

    _lib.require_device()
    return torch.device("cuda:0")
