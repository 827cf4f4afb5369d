mkdir -p gpurun_out/src
for s in C5a C3 C4; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:go_evolve -s 5 -c 1 -o /tmp/p_$s python tools/c2_chunks.py $s 7 > gpurun_out/src/ncu_$s.log 2>&1
  ncu -i /tmp/p_$s.ncu-rep --page source --csv --print-source cuda,sass > /tmp/src_$s.csv 2>/dev/null
  python tools/ncu_lines.py /tmp/src_$s.csv 60 > gpurun_out/src/lines_$s.txt 2>&1
  python tools/ncu_traffic.py /tmp/p_$s.ncu-rep r02b_$s > /dev/null 2>&1; cp profiles/r02b_${s}_ncu_summary.txt gpurun_out/src/ 2>/dev/null
done
