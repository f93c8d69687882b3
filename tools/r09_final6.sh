#!/bin/bash
# evidence after the cooperative-threshold change -> gpurun_out/r09k/
set -u
OUT=gpurun_out/r09k; mkdir -p $OUT
timeout 1700 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "exit $?" >> $OUT/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "exit $?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "exit $?" >> $OUT/bench.err
timeout 2400 python tools/parity_full.py c2 c3 c4 c5 --out $OUT/parity_full.jsonl > $OUT/parity_full.log 2>&1; echo "exit $?" >> $OUT/parity_full.log
timeout 500 python tools/soak.py 300 20261024 > $OUT/soak_oracle.log 2>&1; echo "exit $?" >> $OUT/soak_oracle.log
timeout 300 python tools/soak.py 150 invariance 20261024 > $OUT/soak_invariance.log 2>&1; echo "exit $?" >> $OUT/soak_invariance.log
for f in $OUT/pytest_gpu.log $OUT/smoke.log $OUT/soak_oracle.log $OUT/soak_invariance.log; do tail -n 2 $f; done
grep -o '"config": "c[0-9]"\|"total_mismatches": [0-9]*' $OUT/parity_full.jsonl | paste - -
python -c "import json; d=json.load(open('$OUT/bench.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline'].get('frac_call'), d['e2e']['value'], d['stage_ms'], d['clocks'], d['parity_sample']); print({k: (v.get('gcups'), v.get('ms')) for k, v in d['extra'].items() if isinstance(v, dict)})"
