#!/bin/bash
# Build an alternative libranklab_gpu with extra -D flags for engine tuning:
#   tools/build_variant.sh NAME "-DRL_X=1 -DRL_Y=0"  ->  tools/variants/libNAME.so
set -eu
NAME=$1; FLAGS=${2:-}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=$ROOT/paper_1112_5717_b200/csrc
OUT=$ROOT/tools/variants/build_$NAME
mkdir -p $OUT
ARCH="-gencode arch=compute_100a,code=sm_100a"
pids=()
for f in runtime util gemm_tc bridge trsm_tc panel panel_window trsm perm cup batched tri dist capi; do
  /usr/local/cuda/bin/nvcc $ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr $FLAGS \
    -c -o $OUT/$f.o $SRC/$f.cu &
  pids+=($!)
done
for p in "${pids[@]}"; do wait $p; done
/usr/local/cuda/bin/nvcc $ARCH -shared -o $ROOT/tools/variants/lib$NAME.so $OUT/*.o
echo "tools/variants/lib$NAME.so"
