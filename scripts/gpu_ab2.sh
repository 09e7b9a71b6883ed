#!/bin/bash
# GAT GPU tests on the working-tree library, then the A/B of ab/*.so at C2 (and C5 once).
# usage: scripts/gpu_ab2.sh tag rounds [c5]
cd "$GRAFT_REPO_ROOT"; TAG=${1:-ab}; ROUNDS=${2:-2}; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gat.py tests/test_gpu_gat_dyn.py tests/test_gpu_scale.py tests/test_gpu_dist.py tests/test_gpu_cost.py -q -x -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
tail -3 gpurun_out/pytest_$TAG.log
bash scripts/gpu_ab.sh $TAG $ROUNDS --no-parity --no-ncu
if [ "$3" = "c5" ]; then bash scripts/gpu_ab.sh ${TAG}_c5 1 --no-parity --no-ncu --config c5 --steps 3; fi
echo done
