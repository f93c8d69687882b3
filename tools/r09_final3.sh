#!/bin/bash
# final bench + GPU suite + every-pair parity of c2 / c4 after the last parameter change -> gpurun_out/r09h/
set -u
OUT=gpurun_out/r09h; mkdir -p $OUT
timeout 1700 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "exit $?" >> $OUT/pytest_gpu.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "exit $?" >> $OUT/bench.err
timeout 1200 python tools/parity_full.py c2 c4 --out $OUT/parity_full.jsonl > $OUT/parity_full.log 2>&1; echo "exit $?" >> $OUT/parity_full.log
tail -n 2 $OUT/pytest_gpu.log $OUT/parity_full.log
python -c "import json; d=json.load(open('$OUT/bench.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline'].get('frac_call'), d['e2e']['value'], d['stage_ms'], d['clocks'])"
