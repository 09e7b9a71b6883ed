#!/bin/bash
# Round-end evidence pass: all GPU tests, smoke, the headline bench (+ bf16 gather, c5 in both
# modes), the ncu launch list and one source-correlated ncu --set full of the fused kernels.
# usage: scripts/gpu_round2.sh tag
cd "$GRAFT_REPO_ROOT"; TAG=${1:-r2}; mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 900 python -m pytest tests -m gpu -q --maxfail=30 -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/bench_$TAG.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --gather bf16 > gpurun_out/bench_${TAG}_bf16.log 2>&1
timeout 900 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}_c5.log 2>&1
timeout 900 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --gather bf16 > gpurun_out/bench_${TAG}_c5_bf16.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_ncu_launch_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gat_fwd_ovl|gat_bwd_src_fast" -c 3 -o gpurun_out/prof_$TAG python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/bench_ncu_full_$TAG.log 2>&1
echo done-main
timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__ops_path_tensor_op_utchmma_src_tf32_dst_fp32_sparsity_off.sum.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,launch__grid_size --clock-control none -k regex:gemm_tf32x3 -c 5 --csv --log-file gpurun_out/gemm_$TAG.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/bench_ncu_gemm_$TAG.log 2>&1
echo done-gemm
