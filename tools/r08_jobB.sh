#!/bin/bash
# Full-size parity (every pair of c3, c4, c5 vs the oracle on all host cores), then the bench line.
set -u
OUT=gpurun_out/r08
mkdir -p $OUT
nproc > $OUT/host_cores.txt; free -g >> $OUT/host_cores.txt; grep -m1 "model name" /proc/cpuinfo >> $OUT/host_cores.txt
timeout 2400 python tools/parity_full.py c3 c4 c5 --out $OUT/parity_full.jsonl > $OUT/parity_full.log 2>&1; echo "parity exit $?" >> $OUT/parity_full.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?" >> $OUT/bench.err
tail -c 1500 $OUT/bench.json
