#!/bin/bash
# ncu --set full of the persistent tcgen05 GEMM launches of one C2 step (K1 layer 1, dW, dH).
cd "$GRAFT_REPO_ROOT"; TAG=${1:-g}; mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_tf32x3_persist" -s 5 -c 5 -o gpurun_out/prof_${TAG}_gemm python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-ncu --no-parity > gpurun_out/ncu_${TAG}_gemm.log 2>&1
echo done
