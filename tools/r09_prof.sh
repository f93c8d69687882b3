#!/bin/bash
# ncu launch list of 3 calls on a config + ncu --set full of selected kernels (logs under gpurun_out/r09/)
set -u
OUT=gpurun_out/r09; mkdir -p $OUT
TAG=$1; CFG=$2; KREGEX=$3
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_${TAG}.csv \
  python tools/prof_one.py $CFG > $OUT/launches_${TAG}.log 2>&1
if [ -n "$KREGEX" ]; then
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"$KREGEX" -s 0 -c 4 -o $OUT/ncu_${TAG} -f \
    python tools/prof_one.py $CFG > $OUT/ncu_${TAG}.log 2>&1
fi
python -c "import sys; sys.path.insert(0, \"tools\"); import make_profiles as m; print(m.launch_shares(\"$OUT/launches_${TAG}.csv\"))" | head -30
