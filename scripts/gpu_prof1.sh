#!/bin/bash
# ncu --set full of one launch of kernels matching a regex in the headline step.
# usage: scripts/gpu_prof1.sh tag regex [bench args]
cd "$GRAFT_REPO_ROOT"; TAG=${1:-p}; KRE=$2; shift 2; mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KRE" -c 1 \
  -o gpurun_out/prof_$TAG python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e "$@" > gpurun_out/ncu_$TAG.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_$TAG.log
