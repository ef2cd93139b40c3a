#!/bin/bash
set -u
OUT=gpurun_out/r5a
mkdir -p $OUT
timeout -s KILL 900 ncu --set full --import-source on --clock-control none --warp-sampling-interval 0 \
    -k regex:trsm_node_kernel -c 3 --launch-skip 40 -o $OUT/trsm_node python tools/prof_cup.py 16384 65521 1 > $OUT/ncu_trsm.log 2>&1
timeout -s KILL 900 ncu --set full --import-source on --clock-control none --warp-sampling-interval 0 \
    -k regex:panel_tail_kernel -c 2 --launch-skip 40 -o $OUT/tail python tools/prof_cup.py 16384 65521 1 > $OUT/ncu_tail.log 2>&1
timeout -s KILL 900 ncu --set full --import-source on --clock-control none --warp-sampling-interval 0 \
    -k regex:bridge_kernel -c 2 --launch-skip 20 -o $OUT/bridge python tools/prof_cup.py 16384 65521 1 > $OUT/ncu_bridge.log 2>&1
ls -la $OUT
