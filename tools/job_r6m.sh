#!/bin/bash
set -u
OUT=gpurun_out/${1:-r6m}
bash tools/job_c4.sh $OUT paper_1112_5717_b200/libranklab_gpu.so ${2:-paper_1112_5717_b200/libranklab_gpu.so}
python - > $OUT/trace.txt 2>&1 <<PY
import os, sys
sys.argv = ["prof_c4.py"]
import paper_1112_5717_b200 as G
G.LIB_PATH = os.path.abspath("tools/variants/libb_trace.so")
exec(open("tools/prof_c4.py").read())
PY
