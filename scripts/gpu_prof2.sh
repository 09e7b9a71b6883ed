#!/bin/bash
# ncu --set full of one K2 and one K4f launch of the headline step.  usage: scripts/gpu_prof2.sh tag [bench args]
cd "$GRAFT_REPO_ROOT"; TAG=${1:-p}; shift; mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${NCU_KRE:-gat_fwd_ovl|gat_bwd_src_fast}" -c ${NCU_COUNT:-2} \
  -o gpurun_out/prof_$TAG python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e "$@" > gpurun_out/ncu_$TAG.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_$TAG.log
