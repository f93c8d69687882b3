#!/bin/bash
set -u
OUT=gpurun_out/r08
mkdir -p $OUT
for cfg in c2 c3 c5; do
  for lib in build_var/libsw_xf1.so paper_2208_12350_b200/libsw_b200.so; do
    SW_B200_LIB=$lib timeout 600 python tools/quick_time.py $cfg >> $OUT/ab_h3.log 2>&1
  done
done
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $OUT/pytest_gpu2.log 2>&1; echo "exit $?" >> $OUT/pytest_gpu2.log
grep -E "median|fwd kernel|rev swept|lib:" $OUT/ab_h3.log
tail -n 3 $OUT/pytest_gpu2.log
