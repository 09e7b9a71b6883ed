#!/bin/bash
# bf16-gather pass: its parity tests, the GAT tests, and the headline bench in both gather modes.
cd "$GRAFT_REPO_ROOT"; TAG=${1:-bf}; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gat_bf16.py tests/test_gpu_gat.py -q -x -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --gather bf16 > gpurun_out/bench_${TAG}_bf16.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${TAG}_fp32.log 2>&1
echo done
