#!/bin/bash
# Round-2 correctness job on one B200: compute-sanitizer (4 tools) over tools/sanitize_run.py, then
# the seeded oracle soak (fields + paths, poisoned handle) and the batch-invariance soak.
# Usage: bash tools/r08_sanitize_soak.sh <soak_seconds> <inv_seconds> <seed>
set -u
OUT=gpurun_out/r08
mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
for t in memcheck racecheck synccheck initcheck; do
  extra=""
  [ $t = memcheck ] && extra="--leak-check full"
  timeout 1200 $CS --tool $t $extra --target-processes all --print-limit 50 python tools/sanitize_run.py poison > $OUT/sanitizer_$t.log 2>&1
  echo "exit $?" >> $OUT/sanitizer_$t.log
  tail -3 $OUT/sanitizer_$t.log
done
timeout $(( $1 + 300 )) python tools/soak.py $1 $3 > $OUT/soak_oracle.log 2>&1; echo "exit $?" >> $OUT/soak_oracle.log
timeout $(( $2 + 300 )) python tools/soak.py $2 invariance $3 > $OUT/soak_invariance.log 2>&1; echo "exit $?" >> $OUT/soak_invariance.log
tail -2 $OUT/soak_oracle.log $OUT/soak_invariance.log
