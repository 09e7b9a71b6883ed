#!/bin/bash
# ncu --set full of the EdgeConv K6 / K7 launches (4 layers each) and the GMMConv K8 launches of one step.
cd "$GRAFT_REPO_ROOT"; TAG=${1:-ec}; mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"edgeconv_(fwd|bwd)" -c 8 -o gpurun_out/prof_${TAG}_c3 python bench.py --config edgeconv20 --graph off --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-ncu --no-parity > gpurun_out/ncu_${TAG}_c3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gmm_(fwd|bwd)" -c 6 -o gpurun_out/prof_${TAG}_c4 python bench.py --config monet --graph off --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-ncu --no-parity > gpurun_out/ncu_${TAG}_c4.log 2>&1
echo done
