#!/bin/bash
set -u
OUT=gpurun_out/r2t
mkdir -p $OUT
python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -q -x -p no:cacheprovider -k "not c5_digest" > $OUT/pytest.txt 2>&1; echo rc=$? >> $OUT/pytest.txt
python tools/leaftrace.py tools/variants/liblt.so > $OUT/lt.txt 2>&1
bash tools/job_var.sh $OUT paper_1112_5717_b200/libranklab_gpu.so tools/variants/libnobridge.so
