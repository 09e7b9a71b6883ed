"""GPU: the C++ drop-in (include/gnncg_b200/ops.hpp over the reference's gnncg::Graph /
gnncg::Tensor, linked with the reference's own compiled graph.cpp/tensor.cpp)."""
import os
import subprocess

import pytest

from tests.conftest import ROOT

pytestmark = pytest.mark.gpu
BIN = os.path.join(ROOT, "tests", "cpp", "build", "test_ops_cpp")


def test_cpp_operator_api(cuda):
    assert os.path.exists(BIN), "tests/cpp/build/test_ops_cpp not built (needs /root/reference at build time)"
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    print(r.stdout, r.stderr)
    assert r.returncode == 0 and "OK" in r.stdout
