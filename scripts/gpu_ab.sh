#!/bin/bash
# A/B of library builds on one box: every ab/*.so is copied into place in turn and the
# headline bench runs ROUNDS times alternating.  usage: scripts/gpu_ab.sh tag rounds [bench args]
cd "$GRAFT_REPO_ROOT"; TAG=${1:-ab}; ROUNDS=${2:-2}; shift 2; mkdir -p gpurun_out
LIB=paper_2110_09524_b200/libgnncg_b200.so
cp $LIB gpurun_out/.orig.so
for r in $(seq $ROUNDS); do
  for so in ab/*.so; do
    n=$(basename $so .so); cp $so $LIB
    timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e "$@" > gpurun_out/ab_${TAG}_${n}_$r.log 2>&1
    python - "$n" "$r" gpurun_out/ab_${TAG}_${n}_$r.log >> gpurun_out/ab_${TAG}.txt <<'PY'
import json, sys
n, r, path = sys.argv[1:]
try:
    d = json.loads([l for l in open(path) if l.startswith("{")][-1])
    ks = {k: round(v["ms_per_launch"], 3) for k, v in d["kernels"].items()}
    print(n, r, round(d["ms_per_step"], 3), ks)
except Exception as e:
    print(n, r, "FAILED", e, open(path).read()[-500:])
PY
  done
done
cp gpurun_out/.orig.so $LIB
cat gpurun_out/ab_${TAG}.txt
