#!/bin/bash
# tools/job_var.sh OUTDIR lib1 lib2 ...: C3 timing of library variants on one box
set -u
OUT=$1; shift
mkdir -p $OUT
for v in "$@"; do timeout -s KILL 200 python tools/variant_time.py $v >> $OUT/variants.txt 2>&1; done
