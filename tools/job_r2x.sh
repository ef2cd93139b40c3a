#!/bin/bash
set -u
OUT=gpurun_out/r2x
mkdir -p $OUT
python -m pytest tests -q -x -p no:cacheprovider -m gpu -k "batched or c4" > $OUT/pytest.txt 2>&1; echo rc=$? >> $OUT/pytest.txt
python tools/prof_c4.py > $OUT/c4_new.txt 2>&1
RL_LIB=tools/variants/libbold.so python - > $OUT/c4_old.txt 2>&1 <<'PY'
import os, sys
sys.argv = ["prof_c4.py"]
import paper_1112_5717_b200 as G
G.LIB_PATH = os.path.abspath("tools/variants/libbold.so")
exec(open("tools/prof_c4.py").read())
PY
