#!/bin/bash
# Round-end measurement job (run under gpurun): bench lines, the C3 launch list
# and one ncu --set full capture of the dominant GEMM shape.  Outputs go to
# gpurun_out/prof/ and are copied into profiles/roundN/ by hand.
set -u
OUT=gpurun_out/prof
mkdir -p $OUT
timeout -s KILL 900 python bench.py --steps 5 --warmup 3 > $OUT/bench_c3.json 2> $OUT/bench_c3.err
timeout -s KILL 600 python bench.py --workload c4 --steps 5 --warmup 3 > $OUT/bench_c4.json 2> $OUT/bench_c4.err
timeout -s KILL 600 python bench.py --workload c2 --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_c2.json 2> $OUT/bench_c2.err
timeout -s KILL 600 python bench.py --workload c5 --steps 2 --warmup 2 --no-cpu-baseline > $OUT/bench_c5.json 2> $OUT/bench_c5.err
timeout -s KILL 600 python bench.py --workload c5 --dist --steps 2 --warmup 2 --no-cpu-baseline > $OUT/bench_c5_dist1.json 2> $OUT/bench_c5_dist1.err
timeout -s KILL 600 python tools/prof_dist.py 65536 65521 1024 1024 4096 > $OUT/prof_dist_c5.txt 2>&1
timeout -s KILL 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_c3_reference_arm.json 2> $OUT/bench_ref.err
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches_c3_ncu.csv python tools/prof_cup.py 16384 65521 1 > /dev/null 2>&1
python tools/launch_summary.py $OUT/launches_c3_ncu.csv > $OUT/launches_c3_summary.txt
timeout -s KILL 300 python tools/timeline_cup.py 16384 65521 $OUT/timeline_c3.json > $OUT/timeline_c3.txt 2>&1
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:gemm_tc_kernel \
    -c 1 --launch-skip 1 -o $OUT/gemm_8192 python tools/prof_gemm.py 8192 8192 8192 65521 1 > $OUT/ncu_gemm.log 2>&1
python tools/ncu_json.py $OUT/gemm_8192.ncu-rep gemm_tc_kernel $OUT/gemm_8192_ncu.json \
    "ncu --set full --clock-control none -k regex:gemm_tc_kernel -c 1 --launch-skip 1 python tools/prof_gemm.py 8192 8192 8192 65521 1" > /dev/null
ls -la $OUT
