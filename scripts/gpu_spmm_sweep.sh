#!/bin/bash
# spmm launch-shape sweep (GNNCG_SPMM_OCC x GNNCG_SPMM_NV) on the Reddit-shaped GCN + GCN tests.
cd "$GRAFT_REPO_ROOT"; TAG=${1:-sp}; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gcn.py -q -p no:cacheprovider > gpurun_out/pytest_gcn_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gcn_$TAG.log
GNNCG_SPMM_OCC=8 GNNCG_SPMM_NV=1 timeout 600 python -m pytest tests/test_gpu_gcn.py -q -p no:cacheprovider -k spmm > gpurun_out/pytest_gcn_${TAG}_o8.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gcn_${TAG}_o8.log
for cfg in "4 8" "4 1" "8 1" "8 2" "2 8" "2 1"; do
  set -- $cfg
  GNNCG_SPMM_OCC=$1 GNNCG_SPMM_NV=$2 timeout 300 python bench.py --config gcn --steps 6 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_${TAG}_o$1_nv$2.log 2>&1
done
echo done
