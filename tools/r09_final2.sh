#!/bin/bash
# Round-2 (second session) final validation and evidence on one B200 -> gpurun_out/r09f/
set -u
OUT=gpurun_out/r09g
mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu.txt
timeout 1700 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "exit $?" >> $OUT/pytest_gpu.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "exit $?" >> $OUT/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-extra --no-cpu-baseline > $OUT/launches_bench.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"wavefront_kernel|band_rev_kernel" -s 8 -c 4 \
  -o $OUT/ncu_c4 -f python tools/prof_one.py c4 > $OUT/ncu_c4.log 2>&1
timeout 2400 python tools/parity_full.py c2 c3 c4 c5 --out $OUT/parity_full.jsonl > $OUT/parity_full.log 2>&1; echo "exit $?" >> $OUT/parity_full.log
timeout 800 python tools/soak.py 480 20261021 > $OUT/soak_oracle.log 2>&1; echo "exit $?" >> $OUT/soak_oracle.log
timeout 400 python tools/soak.py 240 invariance 20261021 > $OUT/soak_invariance.log 2>&1; echo "exit $?" >> $OUT/soak_invariance.log
tail -n 2 $OUT/pytest_gpu.log $OUT/parity_full.log $OUT/soak_*.log
python -c "import json; d=json.load(open('$OUT/bench.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline'].get('frac_call'), d['e2e']['value'], d['stage_ms'], d['clocks'])"
