#!/bin/bash
# A/B of an environment switch on one box: bench runs alternate VAR=a / VAR=b.
# usage: scripts/gpu_env_ab.sh tag VAR "a b" rounds [bench args]
cd "$GRAFT_REPO_ROOT"; TAG=$1; VAR=$2; VALS=$3; ROUNDS=${4:-2}; shift 4; mkdir -p gpurun_out
for r in $(seq $ROUNDS); do
  for v in $VALS; do
    env $VAR=$v timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e "$@" > gpurun_out/eab_${TAG}_${v}_$r.log 2>&1
    python - "$VAR=$v" "$r" gpurun_out/eab_${TAG}_${v}_$r.log >> gpurun_out/eab_${TAG}.txt <<'PY'
import json, sys
n, r, path = sys.argv[1:]
try:
    d = json.loads([l for l in open(path) if l.startswith("{")][-1])
    ks = {k: round(v["ms_per_launch"], 3) for k, v in d["kernels"].items()}
    print(n, r, round(d["ms_per_step"], 3), ks)
except Exception as e:
    print(n, r, "FAILED", e, open(path).read()[-800:])
PY
  done
done
cat gpurun_out/eab_${TAG}.txt
