#!/bin/sh
# A/B timing of kernel header sets on the same box: tools/ab_run.sh name[:DEFINE] ...
# (kernel sets under ab_kernels/<name>/, JIT-compiled via GO_KERNEL_DIR)
for round in 1 2; do
  for spec in "$@"; do
    name=${spec%%:*}; def=${spec#*:}; [ "$def" = "$spec" ] && def=GO_JIT_DEFAULT=1
    loops=0; case "$name" in *+loops) loops=1; name=${name%+loops};; esac
    t=$(GO_DEMO_LOOPS=$loops GO_KERNEL_DIR=$PWD/ab_kernels/$name GO_JIT_DEFINE=$def python tools/c2_chunks.py C2 8 2>&1 | tail -n 3 | awk '{s+=$(NF-1)} END {printf "%.2f", s/3}')
    echo "round $round $spec: $t ms/chunk (mean of chunks 6-8)"
  done
done
