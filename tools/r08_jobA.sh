#!/bin/bash
set -u
OUT=gpurun_out/r08
mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
for t in initcheck memcheck; do
  extra=""
  [ $t = memcheck ] && extra="--leak-check full"
  timeout 900 $CS --tool $t $extra --target-processes all --print-limit 50 python tools/sanitize_run.py poison > $OUT/sanitizer2_$t.log 2>&1
  echo "exit $?" >> $OUT/sanitizer2_$t.log
done
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "exit $?" >> $OUT/pytest_gpu.log
bash tools/r08_prof.sh
