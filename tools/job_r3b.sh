#!/bin/bash
# Evidence job: window phase trace, compute-sanitizer (one tool per run) on
# small CUPs, ncu DRAM bytes of the permutation / tail kernels on the
# swap-heavy case s1.
set -u
OUT=gpurun_out/r3b
mkdir -p $OUT
timeout -s KILL 300 python tools/trace_cup.py > $OUT/trace.txt 2>&1
for tool in memcheck racecheck synccheck initcheck; do
  timeout -s KILL 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_cup.py \
      > $OUT/sanitizer_$tool.txt 2>&1; echo "rc=$?" >> $OUT/sanitizer_$tool.txt
done
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed \
    --clock-control none -k regex:"swaps_kernel|compact_kernel|panel_tail_kernel" -c 400 --csv \
    --log-file $OUT/s1_perm_ncu.csv python tools/prof_s1.py 1 > $OUT/s1_ncu.log 2>&1
timeout -s KILL 300 python tools/prof_s1.py 3 > $OUT/s1_time.txt 2>&1
