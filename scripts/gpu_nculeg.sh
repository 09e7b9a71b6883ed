#!/bin/bash
# The bench's in-run ncu DRAM-byte leg on the configs where it failed or mixed launches.
cd "$GRAFT_REPO_ROOT"; TAG=${1:-nl}; mkdir -p gpurun_out
for c in gcn c5 reddit; do
  timeout 1500 python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-parity > gpurun_out/bench_${TAG}_$c.log 2>&1
  grep '^{' gpurun_out/bench_${TAG}_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['ms_per_step'],2), json.dumps(d['roofline'])[:700])"
done
