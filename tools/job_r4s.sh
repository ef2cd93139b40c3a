#!/bin/bash
# Round-2 evidence job: launch list of one warm C3 factorization (tiled), the
# device timeline, ncu --set full of the dominant GEMM shape and of the window
# kernel (fine warp sampling), the batched kernel, the reference arm, and the
# reference's own acceptance suite over the GPU shims run to the end.
set -u
OUT=gpurun_out/r4s
mkdir -p $OUT
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches_c3_ncu.csv python tools/prof_cup.py 16384 65521 1 > /dev/null 2>&1
python tools/launch_summary.py $OUT/launches_c3_ncu.csv > $OUT/launches_c3_summary.txt
timeout -s KILL 300 python tools/timeline_cup.py 16384 65521 $OUT/timeline_c3.json > $OUT/timeline_c3.txt 2>&1
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:gemm_tc_kernel \
    -c 1 --launch-skip 1 -o $OUT/gemm_8192 python tools/prof_gemm.py 8192 8192 8192 65521 1 > $OUT/ncu_gemm.log 2>&1
python tools/ncu_json.py $OUT/gemm_8192.ncu-rep gemm_tc_kernel $OUT/gemm_8192_ncu.json \
    "ncu --set full --clock-control none -k regex:gemm_tc_kernel -c 1 --launch-skip 1 python tools/prof_gemm.py 8192 8192 8192 65521 1" > /dev/null
timeout -s KILL 900 ncu --set full --import-source on --clock-control none --warp-sampling-interval 0 \
    -k regex:panel_window_kernel -c 3 --launch-skip 120 -o $OUT/window python tools/prof_cup.py 16384 65521 1 > $OUT/ncu_window.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none -k regex:cup_batched -c 1 -o $OUT/batched \
    python bench.py --workload c4 --steps 1 --warmup 1 --no-cpu-baseline > $OUT/ncu_batched.log 2>&1
timeout -s KILL 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_reference_arm.json 2> $OUT/bench_ref.err
( cd oracle/_ref && timeout -s KILL 1500 stdbuf -oL ./acceptance_gpu > ../../$OUT/acceptance_gpu_full.txt 2>&1; echo "rc=$?" >> ../../$OUT/acceptance_gpu_full.txt )
ls -la $OUT
