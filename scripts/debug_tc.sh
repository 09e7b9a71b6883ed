#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for d in 0 1 2; do GNNCG_TC_DEBUG=$d timeout 120 python scripts/debug_tc.py; done > gpurun_out/debug_tc.log 2>&1
echo done >> gpurun_out/debug_tc.log
