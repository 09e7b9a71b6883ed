#!/bin/bash
# ncu --set full of the lean K4f (C2) and of K2 / K4f at C5 (DRAM-bound regime).
cd "$GRAFT_REPO_ROOT"; TAG=${1:-p}; mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gat_bwd_src_lean" -c 1 -o gpurun_out/prof_k4_$TAG python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-ncu --no-parity > gpurun_out/ncu_k4_$TAG.log 2>&1
timeout 1500 ncu --set full --clock-control none -k regex:"gat_fwd_lean|gat_bwd_src_lean" -c 2 -o gpurun_out/prof_c5_$TAG python bench.py --config c5 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-ncu --no-parity > gpurun_out/ncu_c5_$TAG.log 2>&1
echo done
