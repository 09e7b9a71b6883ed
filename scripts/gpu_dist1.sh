#!/bin/bash
# Multi-GPU path on one GPU: dist tests (emulated ranks + NCCL world 1), the partitioned bench at world 1.
cd "$GRAFT_REPO_ROOT"; TAG=${1:-d1}; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_graph.py -q -p no:cacheprovider -x > gpurun_out/pytest_dist_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_dist_$TAG.log
timeout 600 python bench.py --partitioned --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_part_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/bench_part_$TAG.log
timeout 900 python bench.py --partitioned --config c5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_part_c5_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/bench_part_c5_$TAG.log
