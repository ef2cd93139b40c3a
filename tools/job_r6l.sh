#!/bin/bash
set -u
OUT=gpurun_out/r6l
mkdir -p $OUT
python - > $OUT/trace.txt 2>&1 <<PY
import os, sys
sys.argv = ["prof_c4.py"]
import paper_1112_5717_b200 as G
G.LIB_PATH = os.path.abspath("tools/variants/libb_trace.so")
exec(open("tools/prof_c4.py").read())
PY
