#!/bin/bash
# ncu --set full of the wavefront kernels on c3 (protein, S16 route) and c5 (multi-stripe S16 + TAG
# short pairs): the third call of tools/prof_one.py (forward then reverse launches).
set -u
OUT=gpurun_out/r08
mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:wavefront_kernel -s 4 -c 2 \
  -o $OUT/ncu_c3 -f python tools/prof_one.py c3 > $OUT/ncu_c3.log 2>&1; echo "c3 exit $?"
timeout 1500 $NCU --set full --clock-control none --import-source on -k regex:wavefront_kernel -s 8 -c 4 \
  -o $OUT/ncu_c5 -f python tools/prof_one.py c5 > $OUT/ncu_c5.log 2>&1; echo "c5 exit $?"
ls -la $OUT
