#!/bin/bash
# ncu --set full (source-correlated) of the first forward K2 launch.  usage: scripts/gpu_k2prof.sh tag [kernel regex]
cd "$GRAFT_REPO_ROOT"; TAG=${1:-k2}; KRE=${2:-gat_fwd}; mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KRE" -c 1 \
  -o gpurun_out/prof_$TAG python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_$TAG.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_$TAG.log
