#!/bin/bash
# EdgeConv kernel variants (ab/*.so): EdgeConv GPU tests under each, then the C3 step A/B at k = 20 and 40.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
LIB=paper_2110_09524_b200/libgnncg_b200.so; cp $LIB gpurun_out/.orig_e.so
for so in ab/*.so; do
  n=$(basename $so .so); cp $so $LIB
  timeout 600 python -m pytest tests/test_gpu_edgeconv_gmm.py tests/test_gpu_models.py -q -x -p no:cacheprovider > gpurun_out/pytest_ec_$n.log 2>&1
  echo "$n pytest rc=$? $(tail -1 gpurun_out/pytest_ec_$n.log)"
done
cp gpurun_out/.orig_e.so $LIB
bash scripts/gpu_ab.sh ec20 2 --config edgeconv20 | tail -0
bash scripts/gpu_ab.sh ec40 2 --config edgeconv40 | tail -0
cat gpurun_out/ab_ec20.txt gpurun_out/ab_ec40.txt
