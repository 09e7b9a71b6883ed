#!/bin/bash
# All GPU tests + the headline bench + the 1B-edge config.  usage: scripts/gpu_check.sh [tag]
cd "$GRAFT_REPO_ROOT"; TAG=${1:-chk}; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --maxfail=30 -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$TAG.log 2>&1
timeout 900 python bench.py --config c5 --steps 3 --warmup 2 --no-e2e > gpurun_out/bench_${TAG}_c5.log 2>&1
echo done
