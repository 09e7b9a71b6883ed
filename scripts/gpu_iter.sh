#!/bin/bash
# Iteration pass: GAT parity tests + headline bench (no CPU baseline).  usage: scripts/gpu_iter.sh tag [extra bench args]
cd "$GRAFT_REPO_ROOT"; TAG=${1:-it}; shift; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gat.py tests/test_gpu_dist.py -q -x -p no:cacheprovider > gpurun_out/pytest_iter_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_iter_$TAG.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/bench_iter_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/bench_iter_$TAG.log
echo done
