#!/bin/bash
# Build an A/B variant of the library: the listed sources recompiled with extra nvcc flags,
# linked with the default build's other objects into ab/<name>.so (for scripts/gpu_ab.sh).
# usage: scripts/build_ab.sh name "extra flags" src.cu [src.cu ...]
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1; FLAGS=$2; shift 2
C=$ROOT/paper_2110_09524_b200/csrc
make -C "$C" -j 8 >/dev/null
T=$(mktemp -d); mkdir -p "$ROOT/ab"
OBJS=""
for o in "$C"/build/*.o; do
  b=$(basename "$o" .o); hit=""
  for s in "$@"; do [ "$(basename "$s" .cu)" = "$b" ] && hit=1; done
  if [ -n "$hit" ]; then
    /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
      -ccbin /usr/bin/g++ -I"$ROOT/include" --expt-relaxed-constexpr -Xptxas -v $FLAGS -c "$C/$b.cu" -o "$T/$b.o" \
      2> "$T/$b.ptxas.log" || (cat "$T/$b.ptxas.log"; exit 1)
    grep -A1 "lean" "$T/$b.ptxas.log" | grep -E "registers|spill" | head -8 || true
    OBJS="$OBJS $T/$b.o"
  else
    OBJS="$OBJS $o"
  fi
done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -ccbin /usr/bin/g++ -o "$ROOT/ab/$NAME.so" $OBJS -ldl
rm -rf "$T"
echo "built ab/$NAME.so"
