#!/bin/bash
# Round-2 first GPU job: C2 launch list + timeline, C3 timeline, sanitizers.
set -u
OUT=gpurun_out/r2a
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt 2>&1
timeout -s KILL 300 python tools/timeline_cup.py c2 65521 $OUT/timeline_c2.json > $OUT/timeline_c2.txt 2>&1
timeout -s KILL 300 python tools/timeline_cup.py 16384 65521 $OUT/timeline_c3.json > $OUT/timeline_c3.txt 2>&1
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches_c2_ncu.csv python tools/prof_c2.py 1 > $OUT/prof_c2.log 2>&1
python tools/launch_summary.py $OUT/launches_c2_ncu.csv > $OUT/launches_c2_summary.txt 2>&1
for tool in memcheck racecheck synccheck; do
  timeout -s KILL 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_cup.py > $OUT/sanitizer_$tool.txt 2>&1
  echo "rc=$?" >> $OUT/sanitizer_$tool.txt
done
ls -la $OUT
