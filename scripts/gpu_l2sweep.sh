#!/bin/bash
# L2 set-aside sweep (bench --l2-persist-mb) at C2 (and C5 once) + the tests the change touches.
cd "$GRAFT_REPO_ROOT"; TAG=${1:-l2s}; ROUNDS=${2:-2}; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_l2.py tests/test_gpu_gat.py tests/test_gpu_cpp.py tests/test_gpu_dist.py -q -x -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
tail -3 gpurun_out/pytest_$TAG.log
for r in $(seq $ROUNDS); do
  for mb in 0 32 48 64; do
    timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-parity --no-ncu --l2-persist-mb $mb > gpurun_out/l2s_${TAG}_${mb}_$r.log 2>&1
    python - "$mb" "$r" gpurun_out/l2s_${TAG}_${mb}_$r.log >> gpurun_out/l2s_${TAG}.txt <<'PY'
import json, sys
n, r, path = sys.argv[1:]
try:
    d = json.loads([l for l in open(path) if l.startswith("{")][-1])
    ks = {k: round(v["ms_per_launch"], 3) for k, v in d["kernels"].items()}
    print("mb=" + n, r, round(d["ms_per_step"], 3), d["config"].get("l2_persist_mb"), ks)
except Exception as e:
    print(n, r, "FAILED", e, open(path).read()[-800:])
PY
  done
done
for mb in 0 48; do
  timeout 900 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-parity --no-ncu --l2-persist-mb $mb > gpurun_out/l2s_${TAG}_c5_$mb.log 2>&1
  grep '^{' gpurun_out/l2s_${TAG}_c5_$mb.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5 mb=$mb', round(d['ms_per_step'],2), {k: round(v['ms_per_launch'],2) for k,v in d['kernels'].items()})" >> gpurun_out/l2s_${TAG}.txt
done
cat gpurun_out/l2s_${TAG}.txt
