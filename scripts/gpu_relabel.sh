#!/bin/bash
# The L2 window under other labellings: generator ids / shuffled / shuffled then degree-relabeled.
cd "$GRAFT_REPO_ROOT"; TAG=${1:-rl}; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_l2.py -q -x -p no:cacheprovider 2>&1 | tail -2
for r in 1 2; do
  for v in "none 48" "random 48" "degree 48" "random 0"; do set -- $v
    timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-parity --no-ncu --relabel $1 --l2-persist-mb $2 > gpurun_out/rl_${TAG}_$1_$2_$r.log 2>&1
    grep "^{" gpurun_out/rl_${TAG}_$1_$2_$r.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('relabel=$1 l2=$2', round(d['ms_per_step'],2), {k: round(v['ms_per_launch'],2) for k,v in d['kernels'].items() if k in ('gat_fwd','gat_bwd_src_fused')})" | tee -a gpurun_out/rl_${TAG}.txt
  done
done
