#!/bin/bash
# last check of the final tree: GPU suite, smoke, bench -> gpurun_out/r09i/
set -u
OUT=gpurun_out/r09i; mkdir -p $OUT
timeout 1700 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "exit $?" >> $OUT/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "exit $?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "exit $?" >> $OUT/bench.err
tail -n 2 $OUT/pytest_gpu.log $OUT/smoke.log
python -c "import json; d=json.load(open('$OUT/bench.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline'].get('frac_call'), d['e2e']['value'], d['stage_ms'], d['clocks'], d['parity_sample'])"
