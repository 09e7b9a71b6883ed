#!/bin/bash
# ncu --set full (source-correlated) of one launch each of the lean K2 and K4f at the headline config.
cd "$GRAFT_REPO_ROOT"; TAG=${1:-p}; mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gat_bwd_src_lean" -c 1 -o gpurun_out/prof_${TAG}_k4f python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-ncu --no-parity > gpurun_out/ncu_${TAG}_k4f.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gat_fwd_lean" -c 1 -o gpurun_out/prof_${TAG}_k2 python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-ncu --no-parity > gpurun_out/ncu_${TAG}_k2.log 2>&1
echo done
