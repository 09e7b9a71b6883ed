#!/bin/bash
# A/B of ab/*.so on the headline config, then one source-correlated ncu --set full of the
# lean K2 / K4f with the default library.  usage: scripts/gpu_abprof.sh tag rounds
cd "$GRAFT_REPO_ROOT"; TAG=${1:-abp}; ROUNDS=${2:-2}; mkdir -p gpurun_out
bash scripts/gpu_ab.sh $TAG $ROUNDS --no-parity --no-ncu
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gat_bwd_src_lean" -c 1 -o gpurun_out/prof_$TAG python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-ncu --no-parity > gpurun_out/bench_ncu_full_$TAG.log 2>&1
echo done
