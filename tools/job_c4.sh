#!/bin/bash
# tools/job_c4.sh OUT lib...: batched parity (default lib) + C4 timing of each lib
set -u
OUT=$1; shift
mkdir -p $OUT
python -m pytest tests -q -x -p no:cacheprovider -m gpu -k "batched or c4" > $OUT/pytest.txt 2>&1; echo rc=$? >> $OUT/pytest.txt
for v in "$@"; do
python - >> $OUT/c4.txt 2>&1 <<PY
import os, sys
sys.argv = ["prof_c4.py"]
import paper_1112_5717_b200 as G
G.LIB_PATH = os.path.abspath("$v")
print("$v")
exec(open("tools/prof_c4.py").read())
PY
done
