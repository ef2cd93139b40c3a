#!/bin/bash
set -u
OUT=gpurun_out/r2m
mkdir -p $OUT
timeout -s KILL 300 python tools/trace_cup.py 16384 65521 > $OUT/trace_c3.txt 2>&1
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:panel_window_kernel -c 1 --launch-skip 130 \
   -o $OUT/window python tools/prof_cup.py 16384 65521 0 > $OUT/ncu_window.log 2>&1
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:panel_tail_kernel -c 1 --launch-skip 130 \
   -o $OUT/tail python tools/prof_cup.py 16384 65521 0 > $OUT/ncu_tail.log 2>&1
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:trsm_node_kernel -c 1 --launch-skip 130 \
   -o $OUT/trsm python tools/prof_cup.py 16384 65521 0 > $OUT/ncu_trsm.log 2>&1
