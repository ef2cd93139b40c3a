#!/bin/bash
set -u
OUT=gpurun_out/r2j
mkdir -p $OUT
timeout -s KILL 300 python tools/debug_threads.py 4 > $OUT/threads.txt 2>&1
RL_NO_PDL=1 timeout -s KILL 300 python tools/debug_threads.py 4 > $OUT/threads_nopdl.txt 2>&1
timeout -s KILL 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -k "not concurrent_host_threads" > $OUT/pytest_gpu.txt 2>&1
echo "rc=$?" >> $OUT/pytest_gpu.txt
for tool in memcheck racecheck synccheck; do
  timeout -s KILL 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_cup.py > $OUT/sanitizer_$tool.txt 2>&1
  echo "rc=$?" >> $OUT/sanitizer_$tool.txt
done
timeout -s KILL 300 python tools/prof_s1.py 2 > $OUT/s1.txt 2>&1
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none --csv \
    -k regex:"swaps_kernel|compact_kernel|panel_tail_kernel" --log-file $OUT/s1_perm_ncu.csv python tools/prof_s1.py 0 > $OUT/s1_ncu.log 2>&1
ls -la $OUT
