#!/bin/bash
# All GPU tests + every BASELINE config line.  usage: scripts/gpu_configs2.sh tag
cd "$GRAFT_REPO_ROOT"; TAG=${1:-cfg}; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --maxfail=30 -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
for c in c5 cora edgeconv20 edgeconv40 monet; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_${TAG}_$c.log 2>&1
done
echo done
