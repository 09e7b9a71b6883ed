#!/bin/bash
# L2 residency-hint sweep (GNNCG_L2_HOT_ROWS) on the Reddit GAT and GCN configs + GCN tests.
cd "$GRAFT_REPO_ROOT"; TAG=${1:-l2}; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gcn.py -q -p no:cacheprovider > gpurun_out/pytest_gcn_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gcn_$TAG.log
for hr in -1 40000 80000 120000; do
  GNNCG_L2_HOT_ROWS=$hr timeout 300 python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_${TAG}_gat_$hr.log 2>&1
  GNNCG_L2_HOT_ROWS=$hr timeout 300 python bench.py --config gcn --steps 6 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_${TAG}_gcn_$hr.log 2>&1
done
echo done
