#!/bin/bash
# Launch lists of the small configs' training steps (CUDA graph off so every kernel is listed):
# only library kernels should appear inside the step.
cd "$GRAFT_REPO_ROOT"; TAG=${1:-sl}; mkdir -p gpurun_out
for c in edgeconv20 monet cora; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${c}_$TAG.csv python bench.py --config $c --steps 2 --warmup 1 --graph off --no-e2e --no-ncu --no-parity --no-cpu-baseline > gpurun_out/bench_ncu_launch_${c}_$TAG.log 2>&1
done
echo done
