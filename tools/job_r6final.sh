#!/bin/bash
# final evidence of this session: full GPU suite, default bench, C4 bench, batched ncu + phase trace
set -u
OUT=gpurun_out/r6final
mkdir -p $OUT
timeout -s KILL 900 python bench.py --steps 5 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err
timeout -s KILL 600 python bench.py --workload c4 --steps 5 --warmup 3 > $OUT/bench_c4.json 2> $OUT/bench_c4.err
timeout -s KILL 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/pytest.txt 2>&1; echo rc=$? >> $OUT/pytest.txt
timeout -s KILL 300 python __graft_entry__.py smoke > $OUT/smoke.txt 2>&1
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:cup_batched_blk -c 1 \
  -o $OUT/batched python tools/prof_c4.py > $OUT/ncu.log 2>&1
python - > $OUT/batched_phase_trace.txt 2>&1 <<PY
import os, sys
sys.argv = ["prof_c4.py"]
import paper_1112_5717_b200 as G
G.LIB_PATH = os.path.abspath("tools/variants/libb_trace.so")
exec(open("tools/prof_c4.py").read())
PY
