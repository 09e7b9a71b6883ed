#!/bin/bash
# Library variants (ab/*.so): the named GPU test files under each, then the step A/B per config.
# usage: scripts/gpu_cfg_ab.sh "tests/a.py tests/b.py" rounds config [config ...]
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out; TESTS=$1; ROUNDS=$2; shift 2
LIB=paper_2110_09524_b200/libgnncg_b200.so; cp $LIB gpurun_out/.orig_c.so
for so in ab/*.so; do
  n=$(basename $so .so); cp $so $LIB
  timeout 600 python -m pytest $TESTS -q -x -p no:cacheprovider > gpurun_out/pytest_cfg_$n.log 2>&1
  echo "$n pytest rc=$? $(tail -1 gpurun_out/pytest_cfg_$n.log)"
done
cp gpurun_out/.orig_c.so $LIB
for c in "$@"; do bash scripts/gpu_ab.sh cfg_$c $ROUNDS --config $c > /dev/null; cat gpurun_out/ab_cfg_$c.txt; done
