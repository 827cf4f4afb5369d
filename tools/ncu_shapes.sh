#!/bin/sh
# ncu captures for profiles/ (one GPU, never multi-rank): the top kernel of each
# BASELINE shape, one launch after warm-up, --set full, summarised on the box
# (tools/ncu_traffic.py -> profiles/<tag>_<shape>_ncu_summary.txt); only the C2
# report is kept (the row reports are ~40 MB each).  Then the launch list of a
# short C2 bench run (per-launch device times: shares, not absolutes).
# Usage: sh tools/ncu_shapes.sh <tag> [shapes]
tag=${1:-r02}
shift
shapes=${*:-C2 C3 C4 C5a C5b}
mkdir -p gpurun_out/profiles
for s in $shapes; do
  timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:go_evolve \
      -s 5 -c 1 -o gpurun_out/${tag}_${s} python tools/c2_chunks.py $s 7 > gpurun_out/ncu_${tag}_${s}.log 2>&1
  extra=""; [ "$s" = "C2" ] && extra="--traffic"
  python tools/ncu_traffic.py gpurun_out/${tag}_${s}.ncu-rep ${tag}_${s} $extra > /dev/null 2>&1
  cp profiles/${tag}_${s}_ncu_summary.txt gpurun_out/profiles/ 2>/dev/null
  [ "$s" = "C2" ] && cp profiles/r02_ncu_traffic.json gpurun_out/profiles/ 2>/dev/null
  [ "$s" = "C2" ] && ncu -i gpurun_out/${tag}_${s}.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${tag}_${s}_source.csv 2>/dev/null
  [ "$s" != "C2" ] && rm -f gpurun_out/${tag}_${s}.ncu-rep
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 3 --warmup 3 \
    --gap-seconds 0 --other-configs 0 --no-cpu-baseline > gpurun_out/ncu_${tag}_launches.log 2>&1
du -sh gpurun_out
