#!/bin/bash
# Opcode histogram of one kernel's SASS in an object / library.  usage: sass_ops.sh file.o kernel_regex
cuobjdump -sass "$1" | awk -v re="$2" '/Function :/{on = ($0 ~ re)} on && /^ +\/\*[0-9a-f]+\*\//{op=$2; if (op ~ /^@/) op=$3; sub(/;$/,"",op); split(op,a,"."); c[a[1]]++; n++} END{printf "total %d\n", n; for (k in c) printf "%5d %s\n", c[k], k}' | sort -k1 -n -r | head -${3:-25}
