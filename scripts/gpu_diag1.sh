cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_graph.py tests/test_gpu_dist.py -q -p no:cacheprovider > gpurun_out/diag1_tests.log 2>&1; echo rc=$? >> gpurun_out/diag1_tests.log
timeout 300 python scripts/diag_nan.py 1e-6 15 auto > gpurun_out/diag_nan_auto.log 2>&1
timeout 300 python scripts/diag_nan.py 1e-6 15 deterministic > gpurun_out/diag_nan_det.log 2>&1
