#!/bin/bash
# All GPU tests, smoke, launch lists of the small configs (library kernels only?), headline bench.
cd "$GRAFT_REPO_ROOT"; TAG=${1:-r02c}; mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 1800 python -m pytest tests -m gpu -q -rs --maxfail=30 -p no:cacheprovider -s > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
for c in edgeconv20 monet; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_${c}_$TAG.csv python bench.py --config $c --steps 2 --warmup 1 --graph off --no-e2e --no-ncu --no-parity > gpurun_out/bench_ncu_launch_${c}_$TAG.log 2>&1
done
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/bench_$TAG.log
echo done
