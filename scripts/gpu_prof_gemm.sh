#!/bin/bash
# New GPU tests + an ncu --set full capture of the tensor-core GEMMs.
cd "$GRAFT_REPO_ROOT"; TAG=${1:-g}; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_dist.py tests/test_gpu_gemm_tc.py -q -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tf32x3 -c 4 -o gpurun_out/prof_gemm_$TAG python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_gemm_$TAG.log 2>&1
echo done
