#!/bin/bash
# GAT GPU tests with ab/<variant>.so in place, then the A/B of all ab/*.so at C2.
# usage: scripts/gpu_abt.sh tag variant rounds [bench args]
cd "$GRAFT_REPO_ROOT"; TAG=$1; VAR=$2; ROUNDS=${3:-2}; shift 3; mkdir -p gpurun_out
LIB=paper_2110_09524_b200/libgnncg_b200.so
cp $LIB gpurun_out/.orig_t.so; cp ab/$VAR.so $LIB
timeout 900 python -m pytest tests/test_gpu_gat.py tests/test_gpu_gat_dyn.py tests/test_gpu_scale.py tests/test_gpu_l2.py tests/test_gpu_cost.py tests/test_gpu_models.py -q -x -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
cp gpurun_out/.orig_t.so $LIB
tail -3 gpurun_out/pytest_$TAG.log
bash scripts/gpu_ab.sh $TAG $ROUNDS --no-parity --no-ncu "$@"
