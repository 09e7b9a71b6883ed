#!/bin/bash
# Bench lines for every BASELINE config (single GPU).  usage: scripts/gpu_configs.sh [tag]
cd "$GRAFT_REPO_ROOT"; TAG=${1:-cfg}; mkdir -p gpurun_out
for c in cora edgeconv20 edgeconv40 monet; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-e2e > gpurun_out/bench_${TAG}_$c.log 2>&1
done
timeout 900 python bench.py --config c5 --steps 3 --warmup 2 --no-e2e > gpurun_out/bench_${TAG}_c5.log 2>&1
echo done
