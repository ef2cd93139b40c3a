#!/bin/bash
set -u
OUT=gpurun_out/r4z
mkdir -p $OUT
for v in paper_1112_5717_b200/libranklab_gpu.so tools/variants/libh1b16.so tools/variants/libh1b32.so tools/variants/libh0b32.so; do
  echo "== $v" >> $OUT/gemm.txt
  for shape in "8192 8192 8192" "16384 1024 15360" "4096 8192 8192"; do
    RL_LIB=$v timeout -s KILL 120 python tools/prof_gemm.py $shape 65521 20 >> $OUT/gemm.txt 2>&1
  done
  RL_LIB=$v timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed \
      --clock-control none -k regex:gemm_tc_kernel -c 1 --launch-skip 1 --csv python tools/prof_gemm.py 8192 8192 8192 65521 1 > $OUT/ncu_$(basename $v .so).csv 2>&1
done
for v in tools/variants/libh1b16.so tools/variants/libh1b32.so; do
  timeout -s KILL 200 python tools/variant_time.py $v >> $OUT/c3.txt 2>&1
  timeout -s KILL 200 python tools/variant_time.py $v 65536 >> $OUT/c5.txt 2>&1
done
timeout -s KILL 200 python tools/variant_time.py paper_1112_5717_b200/libranklab_gpu.so >> $OUT/c3.txt 2>&1
timeout -s KILL 200 python tools/variant_time.py paper_1112_5717_b200/libranklab_gpu.so 65536 >> $OUT/c5.txt 2>&1
