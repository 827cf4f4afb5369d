#!/bin/sh
# ncu captures for profiles/ (one GPU, never multi-rank): the top kernel of each
# BASELINE shape, one launch after warm-up, --set full; and the launch list of a
# short C2 bench run (per-launch device times: shares, not absolutes).
# Usage: sh tools/ncu_shapes.sh <tag> [shapes]      (reports land in gpurun_out/)
tag=${1:-r02}
shift
shapes=${*:-C2 C3 C4 C5a C5b}
mkdir -p gpurun_out
for s in $shapes; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:go_evolve \
      -s 5 -c 1 -o gpurun_out/${tag}_${s} python tools/c2_chunks.py $s 7 > gpurun_out/ncu_${tag}_${s}.log 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 3 --warmup 3 \
    --gap-seconds 0 --other-configs 0 --no-cpu-baseline > gpurun_out/ncu_${tag}_launches.log 2>&1
ls -la gpurun_out/ | grep $tag
