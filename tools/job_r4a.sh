#!/bin/bash
# Re-entry job: full GPU suite, the default bench line, compute-sanitizer
# (one tool per run) and ncu DRAM bytes of the permutation / tail kernels on s1.
set -u
OUT=gpurun_out/r4a
mkdir -p $OUT
nvidia-smi > $OUT/smi.txt 2>&1
timeout -s KILL 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $OUT/pytest.txt 2>&1; echo rc=$? >> $OUT/pytest.txt
timeout -s KILL 900 python bench.py --steps 5 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err
for tool in memcheck racecheck synccheck initcheck; do
  timeout -s KILL 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_cup.py \
      > $OUT/sanitizer_$tool.txt 2>&1; echo "rc=$?" >> $OUT/sanitizer_$tool.txt
done
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed \
    --clock-control none -k regex:"swaps_kernel|compact_kernel|panel_tail_kernel" -c 400 --csv \
    --log-file $OUT/s1_perm_ncu.csv python tools/prof_s1.py 1 > $OUT/s1_ncu.log 2>&1
timeout -s KILL 300 python tools/prof_s1.py 3 > $OUT/s1_time.txt 2>&1
ls -la $OUT
