#!/bin/bash
# Round-2 evidence pass: smoke, all GPU tests, the reference arm then the headline bench
# (the GPU arm reuses the reference arm's full-C2 CPU measurement), the ncu launch list and
# one source-correlated ncu --set full of the fused kernels.
# usage: scripts/gpu_r02.sh tag [skip-tests]
cd "$GRAFT_REPO_ROOT"; TAG=${1:-r2}; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_$TAG.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_$TAG.log
if [ "$2" != "skip-tests" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -rs --maxfail=30 -p no:cacheprovider -s > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
fi
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/bench_ref_$TAG.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/bench_$TAG.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-ncu --no-parity > gpurun_out/bench_ncu_launch_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gat_fwd_lean|gat_bwd_src_lean" -c 3 -o gpurun_out/prof_$TAG python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-ncu --no-parity > gpurun_out/bench_ncu_full_$TAG.log 2>&1
echo done-main
