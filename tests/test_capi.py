"""CPU: the C-ABI library loads, exports every symbol include/gnncg_b200.h declares,
refuses to compute without a B200 (no CPU fallback), and its host-only entry points
(schedule builder, partitioner) satisfy their contracts."""
import ctypes as C
import os
import re

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2110_09524_b200 import _lib
from paper_2110_09524_b200.graph import DeviceSched, partition_rows
from tests.conftest import ROOT


def header_functions():
    src = open(os.path.join(ROOT, "include", "gnncg_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gnncg_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported():
    L = _lib.lib()
    names = header_functions()
    assert len(names) >= 25
    for n in names:
        assert hasattr(L, n), f"{n} declared in gnncg_b200.h but not exported"
    # every binding the Python layer declares is a header function
    assert set(_lib.EXPORTED) <= set(names)
    assert set(names) <= set(_lib.EXPORTED), set(names) - set(_lib.EXPORTED)


def test_version():
    assert b"sm_100a" in _lib.lib().gnncg_version()


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-device path")
def test_no_cpu_fallback():
    L = _lib.lib()
    assert L.gnncg_device_check() == 3  # GNNCG_ERR_NO_DEVICE
    with pytest.raises(_lib.DeviceError):
        _lib.require_device()
    # a compute entry point refuses too
    rc = L.gnncg_gemm(0, 0, 4, 4, 4, None, 4, None, 4, None, 4, None, 0, None)
    assert rc == 3
    assert "no CPU fallback" in _lib.last_error() or "CUDA" in _lib.last_error()


def _sched_reference(off, chunk):
    """Restatement of the schedule contract (runtime.cu:gnncg_sched_build_host)."""
    deg = np.diff(off.astype(np.int64))
    split = [r for r in range(len(deg)) if deg[r] > chunk]
    items = []
    for r in split:
        items += [(r, c) for c in range(-(-deg[r] // chunk))]
    n_split_items = len(items)
    rest = [r for r in range(len(deg)) if deg[r] <= chunk]
    rest.sort(key=lambda r: (-int(np.floor(np.log2(deg[r] + 1))), r))
    items += [(r, 0) for r in rest]
    return items, n_split_items, split


@pytest.mark.parametrize("chunk", [32, 64, 2048])
def test_schedule_builder_contract(chunk):
    rng = np.random.default_rng(chunk)
    deg = np.concatenate([rng.integers(0, 40, 500), [0, 0, 1000, 33, 64, 65, 4097]])
    off = np.concatenate([[0], np.cumsum(deg)]).astype(np.uint64)
    n, ns, nr, items, split_rows, split_first = DeviceSched.host_arrays(off, chunk)
    ref_items, ref_ns, ref_split = _sched_reference(off, chunk)
    assert n == len(ref_items) and ns == ref_ns and nr == len(ref_split)
    assert [tuple(x) for x in items[:2 * n].reshape(-1, 2)] == ref_items
    assert list(split_rows[:nr]) == ref_split
    # every edge covered exactly once by the items' [e0, e1) ranges
    cover = np.zeros(int(off[-1]), np.int32)
    for r, c in ref_items:
        e0 = int(off[r]) + c * chunk
        e1 = min(int(off[r + 1]), e0 + chunk)
        cover[e0:e1] += 1
    assert np.all(cover == 1)
    # split_first delimits each split row's items
    for i, r in enumerate(split_rows[:nr]):
        its = items[2 * split_first[i]:2 * split_first[i + 1]].reshape(-1, 2)
        assert set(its[:, 0]) == {r} and list(its[:, 1]) == list(range(len(its)))


def test_partitioner_matches_oracle():
    rng = np.random.default_rng(1)
    off = np.concatenate([[0], np.cumsum(rng.integers(0, 100, 5000))]).astype(np.uint64)
    for P in (1, 2, 4, 7, 8):
        np.testing.assert_array_equal(partition_rows(off, P), O.partition_rows(off, P))


@pytest.mark.parametrize("w", [0, 1, 22, 32, 1000])
def test_weighted_partitioner_matches_oracle(w):
    """Cost-balanced blocks (edges + w per row) equal the restatement bit for bit; w = 0 is the
    edge-balanced partitioner; a power-law graph's tail rank gets fewer rows as w grows."""
    rng = np.random.default_rng(2)
    deg = (4000.0 / (np.arange(3000) + 5.0)).astype(np.int64) + rng.integers(0, 3, 3000)
    off = np.concatenate([[0], np.cumsum(deg)]).astype(np.uint64)
    for P in (1, 2, 3, 8):
        b = partition_rows(off, P, row_weight=w)
        np.testing.assert_array_equal(b, O.partition_rows_weighted(off, P, w))
        if w == 0:
            np.testing.assert_array_equal(b, partition_rows(off, P))
    if w:
        assert np.diff(partition_rows(off, 8, row_weight=w))[-1] < np.diff(partition_rows(off, 8))[-1]


def test_errors_map_to_reference_exceptions():
    assert issubclass(_lib.GraphError, RuntimeError) and issubclass(_lib.TensorError, RuntimeError)
    with pytest.raises(_lib.ArgumentError):
        _lib.call("gnncg_partition_rows", 10, None, 2, None)


def test_binding_arity_matches_header():
    """Every ctypes signature declares exactly as many arguments as the C prototype."""
    src = open(os.path.join(ROOT, "include", "gnncg_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    protos = dict(re.findall(r"\b(gnncg_[a-z0-9_]+)\s*\(([^)]*)\)\s*;", src))
    for name, (args, _) in _lib._SIGS.items():
        params = protos[name].strip()
        n = 0 if params in ("", "void") else params.count(",") + 1
        assert n == len(args), f"{name}: header has {n} parameters, binding declares {len(args)}"


def test_bench_spawns_one_rank_per_gpu(monkeypatch):
    """`bench.py --gpus N` outside torchrun launches N ranks through torch.distributed.run on
    127.0.0.1 (the driver's N-GPU invocation), passing its own arguments through."""
    import subprocess
    import sys

    import bench

    seen = {}

    class R:
        returncode = 0

    def fake_run(cmd, env=None, **kw):
        seen["cmd"], seen["env"] = cmd, env
        return R()

    monkeypatch.setattr(subprocess, "run", fake_run)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--config", "c5", "--steps", "2"])
    args = bench.parse()
    assert bench.spawn_ranks(args) == 0
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"] and "--nproc-per-node=4" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[-6:] == ["--gpus", "4", "--config", "c5", "--steps", "2"]
    assert seen["env"]["NCCL_DEBUG"] == "INFO"


def _hot_window_reference(off, n):
    """argmax_b off[b+n] - off[b], lowest b on ties (runtime.cu:hot_window_begin)."""
    rows = off.size - 1
    if n <= 0 or n >= rows:
        return 0
    sums = off[n:].astype(np.int64) - off[:rows - n + 1].astype(np.int64)
    return int(np.argmax(sums))


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_hot_window_host(seed):
    rng = np.random.default_rng(seed)
    deg = rng.integers(0, 50, 3000)
    deg[rng.integers(0, 3000, 5)] += 10_000  # a few hubs somewhere
    off = np.concatenate([[0], np.cumsum(deg)]).astype(np.uint64)
    for n in (0, 1, 7, 100, 2999, 3000, 5000):
        assert _lib.hot_window(off, n) == _hot_window_reference(off, n), n
    # degree-descending ids (the Chung-Lu generator): the window starts at row 0
    off = np.concatenate([[0], np.cumsum(np.sort(deg)[::-1])]).astype(np.uint64)
    assert _lib.hot_window(off, 250) == 0
    with pytest.raises(_lib.ArgumentError):
        _lib.call("gnncg_hot_window_host", 10, None, 2, C.byref(_lib.i64()))


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-device path")
def test_l2_persist_needs_device():
    with pytest.raises(_lib.DeviceError):
        _lib.l2_persist(32 << 20)


def test_permute_rows_roundtrip():
    from paper_2110_09524_b200.graph import permute_rows, unpermute_rows

    X = torch.arange(20.0).reshape(10, 2)
    perm = torch.tensor([3, 0, 9, 1, 2, 8, 7, 4, 6, 5])
    Y = permute_rows(X, perm)
    assert torch.equal(Y[0], X[3]) and torch.equal(unpermute_rows(Y, perm), X)
