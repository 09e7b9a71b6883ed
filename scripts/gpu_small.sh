#!/bin/bash
# Model-step tests and the small configs' bench lines + a launch list per config.
cd "$GRAFT_REPO_ROOT"; TAG=${1:-s}; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_models.py tests/test_gpu_edgeconv_gmm.py tests/test_gpu_gcn.py -q -p no:cacheprovider > gpurun_out/pytest_models_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_models_$TAG.log
for c in cora edgeconv20 edgeconv40 monet; do
  timeout 600 python bench.py --config $c --steps 50 --warmup 5 > gpurun_out/bench_${c}_$TAG.log 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${c}_$TAG.csv python bench.py --config $c --steps 2 --warmup 1 --graph off --no-e2e --no-ncu --no-parity > /dev/null 2>&1
done
timeout 900 python bench.py --config c5 --steps 3 --warmup 3 --no-e2e > gpurun_out/bench_c5_$TAG.log 2>&1
timeout 900 python bench.py --gather bf16 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_bf16_$TAG.log 2>&1
echo done
