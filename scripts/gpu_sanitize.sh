#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck) over small-graph GPU tests of the fused kernels,
# the bf16 mode and the tcgen05 GEMM.  usage: scripts/gpu_sanitize.sh tag
cd "$GRAFT_REPO_ROOT"; TAG=${1:-san}; mkdir -p gpurun_out
SEL='tests/test_gpu_gat.py::test_region_forward_and_backward tests/test_gpu_gat.py::test_edgeless_graph tests/test_gpu_gat_bf16.py::test_bf16_region tests/test_gpu_edgeconv_gmm.py tests/test_gpu_gcn.py tests/test_gpu_graph.py'
K='G3 or ER16 or cora or star or edgeless or empty or small or golden'
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 99 --print-limit 20 \
    python -m pytest $SEL -q -x -p no:cacheprovider -k "$K" > gpurun_out/san_${tool}_$TAG.log 2>&1
  echo "rc=$?" >> gpurun_out/san_${tool}_$TAG.log
done
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 99 --print-limit 20 \
  python -m pytest tests/test_gpu_gemm_tc.py -q -x -p no:cacheprovider -k "129 or 300 or identity" > gpurun_out/san_gemm_$TAG.log 2>&1
echo "rc=$?" >> gpurun_out/san_gemm_$TAG.log
# the K6/K7 column widths and K8 (small parametrisations)
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 99 --print-limit 20 \
    python -m pytest tests/test_gpu_edgeconv_gmm.py -q -x -p no:cacheprovider \
    -k "1-64-8-33 or 2-128-10-96 or 2-256-20-128 or 200-1500 or 500-4000 or 12-36 or ragged or 400-6000 or 350-9000" > gpurun_out/san_ecgmm_${tool}_$TAG.log 2>&1
  echo "rc=$?" >> gpurun_out/san_ecgmm_${tool}_$TAG.log
done
# the work-counter item fetch of K2 / K4f forced on small graphs
for tool in memcheck racecheck synccheck; do
  GNNCG_GAT_DYN=2 timeout 900 compute-sanitizer --tool $tool --error-exitcode 99 --print-limit 20 \
    python -m pytest tests/test_gpu_gat.py tests/test_gpu_gat_bf16.py -q -x -p no:cacheprovider \
    -k "G3 or ER16 or cora or edgeless or star" > gpurun_out/san_dyn_${tool}_$TAG.log 2>&1
  echo "rc=$?" >> gpurun_out/san_dyn_${tool}_$TAG.log
done
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 99 --print-limit 20 python -m pytest tests/test_gpu_l2.py -q -x -p no:cacheprovider > gpurun_out/san_l2_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/san_l2_$TAG.log
echo done
