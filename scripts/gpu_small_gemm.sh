#!/bin/bash
# tensor-core vs CUDA-core GEMM on the small configs (GNNCG_GEMM=tc is any value but simt)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for c in edgeconv20 edgeconv40 monet cora; do
  bash scripts/gpu_env_ab.sh $c GNNCG_GEMM "tc simt" 2 --config $c
done
