#!/bin/bash
# ncu --set full with source correlation of the fused GAT kernels (K2 + K4f), one bench step.
# usage: scripts/gpu_src_prof.sh [tag]
cd "$GRAFT_REPO_ROOT"; TAG=${1:-src}; mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gat_fwd_kernel|gat_bwd_src_fast" -c 3 \
  -o gpurun_out/prof_$TAG python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_$TAG.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_$TAG.log
echo done
