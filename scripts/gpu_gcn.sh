#!/bin/bash
# All GPU tests + the headline bench + the GCN config (both gather occupancies).  usage: scripts/gpu_gcn.sh [tag]
cd "$GRAFT_REPO_ROOT"; TAG=${1:-gcn}; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --maxfail=30 -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$TAG.log 2>&1
timeout 600 python bench.py --config gcn --steps 10 --warmup 3 > gpurun_out/bench_${TAG}_gcn.log 2>&1
GNNCG_SPMM_OCC=2 timeout 600 python bench.py --config gcn --steps 10 --warmup 3 --no-e2e > gpurun_out/bench_${TAG}_gcn_occ2.log 2>&1
for c in edgeconv40 monet cora; do timeout 300 python bench.py --config $c --steps 20 --warmup 3 > gpurun_out/bench_${TAG}_$c.log 2>&1; done
echo done
