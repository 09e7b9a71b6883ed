#!/bin/bash
# Round-end evidence, part A: smoke, every GPU test, the reference arm, the headline bench (fp32
# and bf16 gather), every other BASELINE config line, the launch list.  usage: gpu_final.sh tag
cd "$GRAFT_REPO_ROOT"; TAG=${1:-fin}; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/smi_$TAG.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 1500 python -m pytest tests -m gpu -q -rs --maxfail=30 -p no:cacheprovider -s > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/bench_ref_$TAG.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/bench_$TAG.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --gather bf16 > gpurun_out/bench_${TAG}_bf16.log 2>&1
for c in c5 cora edgeconv20 edgeconv40 monet gcn; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_${TAG}_$c.log 2>&1
done
timeout 900 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --gather bf16 > gpurun_out/bench_${TAG}_c5_bf16.log 2>&1
timeout 900 python bench.py --partitioned --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-ncu > gpurun_out/bench_${TAG}_partitioned.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-ncu --no-parity > gpurun_out/bench_ncu_launch_$TAG.log 2>&1
echo done
