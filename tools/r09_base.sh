#!/bin/bash
# Round-2 session-2 baseline: GPU tests + quick timings of c2/c3/c5 (logs under gpurun_out/r09/).
set -u
OUT=gpurun_out/r09
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt
for c in c2 c3; do timeout 600 python tools/quick_time.py $c > $OUT/base_$c.log 2>&1; done
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $OUT/pytest_gpu_base.log 2>&1; echo "exit $?" >> $OUT/pytest_gpu_base.log
tail -n 3 $OUT/pytest_gpu_base.log; grep -h -E "median|fwd kernel|rev swept" $OUT/base_*.log
