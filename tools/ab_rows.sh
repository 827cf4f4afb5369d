#!/bin/sh
# Row-kernel A/B on one box: this tree vs the tree under $1 (a built worktree)
# for the BASELINE row shapes; mean of the last 3 of 7 chunks.
for round in 1 2; do
  for c in ${SHAPES:-C3 C4 C5a C5b C1}; do
    a=$(python tools/c2_chunks.py $c 7 2>&1 | tail -n 3 | awk '{s+=$(NF-1)} END {printf "%.2f", s/3}')
    b=$(cd "$1" && python tools/c2_chunks.py $c 7 2>&1 | tail -n 3 | awk '{s+=$(NF-1)} END {printf "%.2f", s/3}')
    echo "round $round $c: cur $a ms  base $b ms"
  done
done
