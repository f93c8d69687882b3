#!/bin/bash
# Round-2 final validation and evidence on one B200 (all logs under gpurun_out/r08f/).
set -u
OUT=gpurun_out/r08f
mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
NCU=/usr/local/cuda/bin/ncu
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "exit $?" >> $OUT/pytest_gpu.log
for t in memcheck racecheck synccheck initcheck; do
  extra=""; [ $t = memcheck ] && extra="--leak-check full"
  timeout 900 $CS --tool $t $extra --target-processes all --print-limit 30 python tools/sanitize_run.py poison > $OUT/sanitizer_$t.log 2>&1
  echo "exit $?" >> $OUT/sanitizer_$t.log
done
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_r08.csv \
  python bench.py --steps 2 --warmup 3 --no-extra --no-cpu-baseline > $OUT/launches_bench.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:wavefront_kernel -s 4 -c 2 -o $OUT/ncu_c4 -f \
  python tools/prof_one.py c4 > $OUT/ncu_c4.log 2>&1
timeout 2400 python tools/parity_full.py c3 c4 c5 --out $OUT/parity_full.jsonl > $OUT/parity_full.log 2>&1; echo "exit $?" >> $OUT/parity_full.log
timeout 1100 python tools/soak.py 900 20261018 > $OUT/soak_oracle.log 2>&1; echo "exit $?" >> $OUT/soak_oracle.log
timeout 500 python tools/soak.py 300 invariance 20261018 > $OUT/soak_invariance.log 2>&1; echo "exit $?" >> $OUT/soak_invariance.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "exit $?" >> $OUT/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
tail -n 2 $OUT/pytest_gpu.log $OUT/parity_full.log $OUT/soak_*.log
