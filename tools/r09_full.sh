#!/bin/bash
# full GPU test suite + bench (default contract run) -> gpurun_out/r09/
set -u
OUT=gpurun_out/r09; mkdir -p $OUT
TAG=$1
timeout 1700 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/pytest_full_$TAG.log 2>&1; echo "exit $?" >> $OUT/pytest_full_$TAG.log
tail -n 3 $OUT/pytest_full_$TAG.log
timeout 900 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "exit $?" >> $OUT/bench_$TAG.err
python -c "import json; d=json.load(open('$OUT/bench_$TAG.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline'].get('frac_call'), d['e2e']['value'], d['stage_ms']); print({k: (v.get('gcups'), v.get('ms')) for k, v in d.get('extra', {}).items() if isinstance(v, dict)})" 2>&1 | tail -3
tail -3 $OUT/bench_$TAG.err
