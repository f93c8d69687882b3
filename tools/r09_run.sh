#!/bin/bash
# usage: bash tools/r09_run.sh TAG "pytest -k expr" "cfgs..."  (logs under gpurun_out/r09/)
set -u
OUT=gpurun_out/r09; mkdir -p $OUT
TAG=$1; KEXPR=$2; CFGS=$3
if [ -n "$KEXPR" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "$KEXPR" > $OUT/pytest_$TAG.log 2>&1; echo "exit $?" >> $OUT/pytest_$TAG.log
  tail -n 3 $OUT/pytest_$TAG.log
fi
for c in $CFGS; do timeout 900 python tools/quick_time.py $c > $OUT/time_${TAG}_$c.log 2>&1; grep -h -E "median|fwd kernel|rev swept|stages" $OUT/time_${TAG}_$c.log; done
