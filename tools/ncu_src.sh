#!/bin/sh
# ncu source-line profiles of the row shapes (one GPU): --set full of one evolve
# launch after warm-up, aggregated on the box by tools/ncu_lines.py; summaries
# and top lines land in gpurun_out/src/.  Usage: sh tools/ncu_src.sh <tag> [shapes]
tag=${1:-r02b}
shift
shapes=${*:-C5a C3 C4}
mkdir -p gpurun_out/src
for s in $shapes; do
  timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:go_evolve -s 5 -c 1 -o /tmp/p_$s python tools/c2_chunks.py $s 7 > gpurun_out/src/ncu_$s.log 2>&1
  ncu -i /tmp/p_$s.ncu-rep --page source --csv --print-source cuda,sass > /tmp/src_$s.csv 2>/dev/null
  python tools/ncu_lines.py /tmp/src_$s.csv 60 > gpurun_out/src/${tag}_lines_$s.txt 2>&1
  python tools/ncu_traffic.py /tmp/p_$s.ncu-rep ${tag}_$s > /dev/null 2>&1; cp profiles/${tag}_${s}_ncu_summary.txt gpurun_out/src/ 2>/dev/null
done
